"""Randomised parity: random geometries, layouts, cache memory kinds, block
tables, movers, launch shapes and the resident engine -- every pull
bit-exact against the oracle, with the in-kernel bounds audit on (zero
violations).  Seeded, so failures reproduce."""
import os
import random

import numpy as np
import pytest
import torch

import kvdgen
from gpu_helpers import (assert_layers_equal, cache_for, make_pair, next_request_id,
                         pull_and_wait)
from oracle import oracle
from paper_2501_14743_b200 import kvd

pytestmark = pytest.mark.gpu


def _geom(rng):
    dt = rng.choice([kvdgen.FP16, kvdgen.BF16, kvdgen.FP8, kvdgen.FP32])
    e = kvdgen.ELEM_BYTES[dt]
    while True:
        H = rng.choice([1, 2, 3, 4, 8])
        D = rng.choice([8, 16, 32, 64, 128])
        L = rng.choice([1, 2, 4, 8, 16, 32])
        if (L * H * D * e) % 16 == 0:
            break
    NL = rng.randint(1, 4)
    NB = rng.randint(4, 160)
    sub = L * H * D
    kind = rng.choice(["default", "block_major", "padded_major", "padded_outer"])
    pad = 16 // e if 16 % e == 0 else 16
    if kind == "default":
        stride = (0,) * 5
    elif kind == "block_major":
        stride = (2 * sub, sub, H * D, D, 1)
    elif kind == "padded_major":
        stride = (2 * sub + pad * rng.randint(1, 4), sub, H * D, D, 1)
    else:
        sb = sub + pad * rng.randint(1, 3)
        stride = (sb, NB * sb + pad, H * D, D, 1)
    return kvdgen.CacheGeom(NL, H, D, L, NB, dt, stride)


def _opts(rng):
    v = rng.choice([kvd.VARIANT_AUTO, kvd.VARIANT_LSU, kvd.VARIANT_LSU32, kvd.VARIANT_TMA])
    o = {kvd.OPT_VARIANT: v}
    if rng.random() < 0.6:
        o[kvd.OPT_TILE_BYTES] = 512 * rng.choice([1, 2, 3, 8, 16, 32])
    if v == kvd.VARIANT_TMA:
        o[kvd.OPT_THREADS] = 32 * rng.choice([1, 2, 4])
        o[kvd.OPT_STAGES] = rng.choice([2, 3, 4])
        o[kvd.OPT_TILE_BYTES] = min(o.get(kvd.OPT_TILE_BYTES, 4096), 16384)
        # the ring (pipes x stages x tile) must fit 225 KiB of shared memory,
        # else kvd_pull refuses it with KVD_EINVAL (tested in test_gpu_parity)
        while (o[kvd.OPT_THREADS] // 32) * o[kvd.OPT_STAGES] * o[kvd.OPT_TILE_BYTES] > 225 * 1024:
            o[kvd.OPT_TILE_BYTES] //= 2
    elif rng.random() < 0.5:
        o[kvd.OPT_THREADS] = 32 * rng.choice([1, 4, 8, 16])
    if rng.random() < 0.3:
        o[kvd.OPT_MAX_CTAS] = rng.randint(1, 9)
    if rng.random() < 0.2:
        o[kvd.OPT_COALESCE] = 0
    if rng.random() < 0.3:
        o[kvd.OPT_EARLY_LOADS] = rng.choice([0, 1, 3, 8])   # (over NVLink) source reads early
    if rng.random() < 0.25:
        o[kvd.OPT_STREAMS] = 2                     # library streams (completion via wait)
    elif v == kvd.VARIANT_AUTO and rng.random() < 0.3:
        # the resident engine takes the short requests (<= 2 MiB, <= 64 runs);
        # the rest still launch, interleaved with the posted ones
        o[kvd.OPT_ENGINE] = rng.choice([1, 2, 4, 8, 16])
    return o


# KVD_FUZZ_SEEDS=N widens the sweep (a 3000-seed soak ran once)
@pytest.mark.parametrize("seed", range(int(os.environ.get("KVD_FUZZ_SEEDS", "200"))))
def test_fuzz_pull(seed):
    rng = random.Random(seed)
    g = _geom(rng)
    dg = g.with_blocks(g.num_blocks + rng.randint(0, 20)) if not any(g.stride) else g
    # caches in torch memory, one allocation per layer or one for all layers,
    # or in exportable VMM memory (kvd_mem_alloc, §8 f3 groundwork)
    mem = rng.choice(["torch", "torch", "torch", "single", "vmm"])
    # on boxes with two GPUs half the cases pull over NVLink (GPU1 <- GPU0:
    # the TMA ring, early reads and tile claiming of the auto policy)
    over_link = rng.random() < 0.5 and torch.cuda.device_count() > 1
    pair = make_pair(g, dg, seed=1000 + seed, single_allocation=mem == "single",
                     src_memory="vmm" if mem == "vmm" else "torch",
                     dst_memory="vmm" if mem == "vmm" else "torch",
                     src_dev=0, dst_dev=1 if over_link else 0)
    try:
        pair.peer.set(kvd.OPT_AUDIT, 1)
        opts = _opts(rng)
        for k, v in opts.items():
            pair.peer.set(k, v)
        rev = None          # the push side (§8 f2): local = prefill cache, imported = decode cache
        pulled = []         # request ids the prefill side must see released (pulls only)
        exp = pair.dst_host
        for it in range(3):
            n = rng.randint(0, min(g.num_blocks, dg.num_blocks))
            kind = rng.choice(["random", "fragmented", "contiguous"])
            if kind == "random" or n == 0:
                s, d = kvdgen.random_table(n, g.num_blocks, dg.num_blocks, seed=seed * 10 + it)
            elif kind == "fragmented":
                s, d = kvdgen.fragmented_table(n, g.num_blocks, dg.num_blocks, seed=seed * 10 + it)
            else:
                s, d = kvdgen.contiguous_table(n, rng.randint(0, g.num_blocks - n),
                                               rng.randint(0, dg.num_blocks - n))
            op = rng.random()
            if op < 0.15:                              # push the same table instead
                if rev is None:
                    rev = pair.src.open_peer(pair.dst.export())
                    rev.set(kvd.OPT_AUDIT, 1)
                    for k, v in opts.items():
                        if k != kvd.OPT_ENGINE:        # the engine pulls only
                            rev.set(k, v)
                rid = next_request_id()
                rev.push(rid, s, d)
                rev.wait(rid)
            elif op < 0.4 and n > 1:                   # batched drain of 2-3 requests
                cut = sorted(rng.sample(range(1, n), min(2, n - 1)))
                parts = np.split(np.arange(n), cut)
                tables = [(s[p], d[p]) for p in parts]
                rids = [next_request_id() for _ in tables]
                pair.peer.pull_batch(rids, tables)
                for r in rids:
                    pair.peer.wait(r)
                pulled += rids
            else:
                rid = next_request_id()
                pull_and_wait(pair, s, d, request_id=rid)
                pulled.append(rid)
            exp = pair.expected(s, d, exp)
        assert pair.peer.audit() == 0
        if rev is not None:
            assert rev.audit() == 0
        # Complete() reached the prefill side once per pulled request
        assert sorted(pair.src.poll_released()) == sorted(pulled)
        assert_layers_equal(pair.download_dst(), exp)
    finally:
        if rev is not None:
            rev.close()
        pair.close()


# options a serving loop may change between requests while others are in flight
_LIVE_OPTS = [(kvd.OPT_STREAMS, [0, 2, 4]), (kvd.OPT_ENGINE, [0, 4, 16]),
              (kvd.OPT_TIMING, [0, 2]), (kvd.OPT_EARLY_LOADS, [0, 2, 8]),
              (kvd.OPT_COALESCE, [0, 1]), (kvd.OPT_VARIANT, [kvd.VARIANT_AUTO, kvd.VARIANT_LSU32,
                                                             kvd.VARIANT_TMA]),
              (kvd.OPT_MAX_CTAS, [0, 3, 64])]


@pytest.mark.parametrize("seed", range(int(os.environ.get("KVD_FUZZ_SEEDS", "200")) // 4))
def test_fuzz_live_sequence(seed):
    """A random serving sequence on one peer: single pulls and batched drains
    left in flight, options changed in between (library streams, the resident
    engine, timing, early reads, coalescing, mover, grid), completions
    retired with kvd_poll_many at random points.  Destinations are disjoint
    across the sequence, so the result is order-free: the whole cache must
    equal the oracle with every table applied, and the prefill side must see
    exactly the pulled request ids released."""
    rng = random.Random(10_000 + seed)
    g = kvdgen.CacheGeom(rng.randint(1, 3), rng.choice([1, 2, 4]), rng.choice([32, 64, 128]),
                         rng.choice([8, 16]), 2048, rng.choice([kvdgen.FP16, kvdgen.BF16]))
    over_link = rng.random() < 0.5 and torch.cuda.device_count() > 1
    pair = make_pair(g, g, seed=5000 + seed, dst_dev=1 if over_link else 0)
    try:
        sizes = [rng.choice([1, 2, 5, 16, 40, 120]) for _ in range(48)]
        while sum(sizes) > 1500:
            sizes.pop()
        tables = kvdgen.disjoint_fragmented_tables(sizes, 2048, 2048, seed=seed)
        pending, pulled, k = set(), [], 0
        exp = pair.dst_host
        while k < len(tables):
            op = rng.random()
            if op < 0.2:
                opt, vals = rng.choice(_LIVE_OPTS)
                pair.peer.set(opt, rng.choice(vals))
                continue
            if op < 0.3 and pending:
                pending -= set(pair.peer.poll_many(sorted(pending)))
                continue
            if op < 0.45 and k + 1 < len(tables):
                m = min(len(tables) - k, rng.randint(2, 4))
                rids = [next_request_id() for _ in range(m)]
                pair.peer.pull_batch(rids, tables[k:k + m])
                batch = tables[k:k + m]
                k += m
            else:
                rids = [next_request_id()]
                pair.peer.pull(rids[0], *tables[k])
                batch = [tables[k]]
                k += 1
            pending.update(rids)
            pulled += rids
            for s, d in batch:
                exp = pair.expected(s, d, exp)
        for r in sorted(pending):
            pair.peer.wait(r)
        assert_layers_equal(pair.download_dst(), exp)
        assert sorted(pair.src.poll_released()) == sorted(pulled)
    finally:
        pair.close()


@pytest.mark.parametrize("seed", range(int(os.environ.get("KVD_FUZZ_SEEDS", "200")) // 10))
def test_fuzz_two_exporters_one_decode_cache(seed):
    """Two prefill caches (one over NVLink on 2-GPU boxes) feed ONE decode
    cache through two peers whose options -- resident engine, library
    streams, mover -- are drawn independently, requests interleaved at
    random and left in flight: per-peer slots, engines and release mailboxes
    stay separate (each exporter sees exactly its own request ids), and the
    decode cache equals the oracle with every table applied."""
    rng = random.Random(20_000 + seed)
    g = kvdgen.CacheGeom(2, 2, 64, 16, 1024, kvdgen.FP16)
    two = torch.cuda.device_count() > 1
    srcs = [cache_for(g, 0), cache_for(g, 1 if two and rng.random() < 0.7 else 0)]
    dst = cache_for(g, 0)
    hosts = []
    for i, c in enumerate(srcs + [dst]):
        h = [kvdgen.random_bytes(c.layer_bytes, 7000 + 31 * seed + 7 * i + l)
             for l in range(g.num_layers)]
        for t, b in zip(c.layers, h):
            t.copy_(torch.from_numpy(b))
        hosts.append(h)
    for c in srcs + [dst]:
        torch.cuda.synchronize(c.device)
    peers = [dst.open_peer(c.export()) for c in srcs]
    try:
        for p in peers:
            p.set(kvd.OPT_ENGINE, rng.choice([0, 4, 16]))
            if rng.random() < 0.3:
                p.set(kvd.OPT_STREAMS, 2)
            p.set(kvd.OPT_VARIANT, rng.choice([kvd.VARIANT_AUTO, kvd.VARIANT_AUTO,
                                               kvd.VARIANT_LSU32, kvd.VARIANT_TMA]))
        sizes = [rng.choice([1, 3, 8, 24]) for _ in range(40)]
        tables = kvdgen.disjoint_fragmented_tables(sizes, 1024, 1024, seed=seed)
        exp = [d.copy() for d in hosts[2]]
        pulled, inflight = ([], []), []
        for s, d in tables:
            i = rng.randrange(2)
            rid = next_request_id()
            peers[i].pull(rid, s, d)
            pulled[i].append(rid)
            inflight.append((i, rid))
            rc = oracle.pull(hosts[i], g.stride, g.num_blocks, exp, g.stride, g.num_blocks,
                             g.num_kv_heads, g.head_dim, g.block_size, g.elem_bytes, s, d)
            assert rc == oracle.OK
            if rng.random() < 0.2:
                for j, r in inflight:
                    peers[j].wait(r)
                inflight = []
        for j, r in inflight:
            peers[j].wait(r)
        torch.cuda.synchronize(dst.device)
        assert_layers_equal([t.cpu().numpy() for t in dst.layers], exp)
        for i in range(2):
            assert sorted(srcs[i].poll_released()) == sorted(pulled[i])
    finally:
        for p in peers:
            p.close()
        for c in srcs + [dst]:
            c.close()
