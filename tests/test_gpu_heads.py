"""§8 f4 -- TP-resharding pulls: decode shard j of a TP=4 decode group pulls
prefill TP=8 shards 2j and 2j+1 into its two head slices.  Expected bytes
come from the oracle's head-offset element loop (oracle_pull_heads)."""
import os
import random

import numpy as np
import pytest
import torch

import kvdgen
from gpu_helpers import assert_layers_equal, cache_for, next_request_id
from oracle import oracle
from paper_2501_14743_b200 import kvd

pytestmark = pytest.mark.gpu


def _fill(cache, seed):
    host = [kvdgen.random_bytes(cache.layer_bytes, seed + l) for l in range(len(cache.layers))]
    for t, h in zip(cache.layers, host):
        t.copy_(torch.from_numpy(h))
    return host


def _run(src_dev, dst_dev, nl=4, nb=64, hs=1, hd=2, d=128, n=40, batch=False, seed=0,
         variant=None, audit=False):
    shards = [cache_for(kvdgen.CacheGeom(nl, hs, d, 16, nb, kvdgen.BF16), src_dev)
              for _ in range(hd // hs)]
    dst = cache_for(kvdgen.CacheGeom(nl, hd, d, 16, nb, kvdgen.BF16), dst_dev)
    hosts = [_fill(c, 1000 * (i + 1) + seed) for i, c in enumerate(shards)]
    expected = _fill(dst, 99 + seed)
    torch.cuda.synchronize(src_dev)
    torch.cuda.synchronize(dst_dev)
    peers = [dst.open_peer_heads(c.export(), i * hs) for i, c in enumerate(shards)]
    for p in peers:
        if variant is not None:
            p.set(kvd.OPT_VARIANT, variant)
        if audit:
            p.set(kvd.OPT_AUDIT, 1)
    s_ids, d_ids = kvdgen.fragmented_table(n, nb, nb, seed=seed + 3)
    try:
        for i, p in enumerate(peers):
            if batch:
                half = n // 2
                rids = [next_request_id(), next_request_id()]
                p.pull_batch(rids, [(s_ids[:half], d_ids[:half]), (s_ids[half:], d_ids[half:])])
                for r in rids:
                    p.wait(r)
            else:
                rid = next_request_id()
                p.pull(rid, s_ids, d_ids)
                p.wait(rid)
                assert p.info()["bytes"] == n * nl * 2 * 16 * hs * d * 2
            rc = oracle.pull_heads(hosts[i], (0,) * 5, nb, hs, expected, (0,) * 5, nb, hd, i * hs,
                                   d, 16, 2, s_ids, d_ids)
            assert rc == oracle.OK
        torch.cuda.synchronize(dst_dev)
        assert_layers_equal([t.cpu().numpy() for t in dst.layers], expected)
        if audit:
            assert all(p.audit() == 0 for p in peers)
        return [p.info() for p in peers]
    finally:
        for p in peers:
            p.close()
        dst.close()
        for c in shards:
            c.close()


@pytest.mark.parametrize("hs,hd", [(1, 2), (2, 8), (4, 8), (1, 4)])
def test_tp_resharding_loopback(hs, hd):
    _run(0, 0, hs=hs, hd=hd, seed=hs * 10 + hd)


def test_tp_resharding_batched():
    _run(0, 0, batch=True, seed=5)


def test_head_slice_rejects_bad_offsets():
    src = cache_for(kvdgen.CacheGeom(2, 2, 128, 16, 8, kvdgen.BF16), 0)
    dst = cache_for(kvdgen.CacheGeom(2, 3, 128, 16, 8, kvdgen.BF16), 0)
    try:
        with pytest.raises(kvd.KvdError) as ei:
            dst.open_peer_heads(src.export(), 2)          # heads 2..3 of 3
        assert ei.value.status == kvd.ELAYOUT
        with pytest.raises(kvd.KvdError) as ei:
            dst.open_peer(src.export())                   # plain pair: heads must match
        assert ei.value.status == kvd.ELAYOUT
        p = dst.open_peer_heads(src.export(), 1)
        rev = src.open_peer(src.export())
        rev.close()
        with pytest.raises(kvd.KvdError):
            p.push(next_request_id(), [0], [1])           # no push on a head-sliced peer
        p.close()
    finally:
        dst.close()
        src.close()


@pytest.mark.gpu2
def test_tp_resharding_two_gpus_70b_shapes():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    infos = _run(0, 1, nl=80, nb=600, hs=1, hd=2, n=512, seed=7, audit=True)
    assert all(i["variant"] == kvd.VARIANT_LSU for i in infos)   # AUTO: LSU for head slices
    infos = _run(0, 1, nl=80, nb=600, hs=1, hd=2, n=512, seed=8, audit=True,
                 variant=kvd.VARIANT_TMA)                        # the TMA head mover over NVLink
    assert all(i["variant"] == kvd.VARIANT_TMA for i in infos)


@pytest.mark.parametrize("hs,hd,nl", [(1, 2, 4), (2, 8, 3), (4, 8, 2), (1, 4, 5)])
@pytest.mark.parametrize("batch", [False, True])
def test_tp_resharding_tma_rows(hs, hd, nl, batch):
    """The TMA head-slice mover (bulk loads of whole remote units, warp-wide
    strided row stores) forced on one GPU, audited; single pulls and batches."""
    infos = _run(0, 0, nl=nl, hs=hs, hd=hd, n=37, batch=batch, seed=hs * 10 + hd,
                 variant=kvd.VARIANT_TMA, audit=True)
    if not batch:
        assert all(i["variant"] == kvd.VARIANT_TMA for i in infos)


# KVD_FUZZ_SEEDS widens it like tests/test_gpu_fuzz.py
@pytest.mark.parametrize("seed", range(int(os.environ.get("KVD_FUZZ_SEEDS", "60"))))
def test_head_slice_fuzz(seed):
    """Random head-slice pulls (§8 f4): shapes, dtypes, block sizes, head
    offsets, tables, movers (AUTO / LSU / TMA rows) and ring shapes, single
    or batched, over NVLink half the time on 2-GPU boxes, bounds audit on --
    bit-exact against the oracle's head-offset element loop."""
    rng = random.Random(seed)
    dt = rng.choice([kvdgen.FP16, kvdgen.BF16, kvdgen.FP8, kvdgen.FP32])
    e = kvdgen.ELEM_BYTES[dt]
    nl, d, bs = rng.randint(1, 4), rng.choice([32, 64, 128]), rng.choice([4, 8, 16])
    hs = rng.choice([1, 2])
    hd = hs * rng.choice([1, 2, 3, 4])
    off = rng.randrange(0, hd - hs + 1)
    nb_s, nb_d = rng.randint(8, 96), rng.randint(8, 96)
    over_link = rng.random() < 0.5 and torch.cuda.device_count() > 1
    src = cache_for(kvdgen.CacheGeom(nl, hs, d, bs, nb_s, dt), 0)
    dst = cache_for(kvdgen.CacheGeom(nl, hd, d, bs, nb_d, dt), 1 if over_link else 0)
    try:
        host = _fill(src, 500 + seed)
        expected = _fill(dst, 900 + seed)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(dst.device)
        p = dst.open_peer_heads(src.export(), off)
        p.set(kvd.OPT_AUDIT, 1)
        v = rng.choice([kvd.VARIANT_AUTO, kvd.VARIANT_LSU, kvd.VARIANT_TMA])
        p.set(kvd.OPT_VARIANT, v)
        if v == kvd.VARIANT_TMA and rng.random() < 0.5:
            p.set(kvd.OPT_THREADS, 32 * rng.choice([1, 2, 4]))
            p.set(kvd.OPT_STAGES, rng.choice([2, 3]))
        try:
            for it in range(3):
                n = rng.randint(0, min(nb_s, nb_d))
                table = kvdgen.random_table if rng.random() < 0.5 else kvdgen.fragmented_table
                s_ids, d_ids = table(n, nb_s, nb_d, seed=seed * 10 + it)
                if n > 1 and rng.random() < 0.3:
                    cut = rng.randrange(1, n)
                    rids = [next_request_id(), next_request_id()]
                    p.pull_batch(rids, [(s_ids[:cut], d_ids[:cut]), (s_ids[cut:], d_ids[cut:])])
                    for r in rids:
                        p.wait(r)
                else:
                    rid = next_request_id()
                    p.pull(rid, s_ids, d_ids)
                    p.wait(rid)
                rc = oracle.pull_heads(host, (0,) * 5, nb_s, hs, expected, (0,) * 5, nb_d, hd, off,
                                       d, bs, e, s_ids, d_ids)
                assert rc == oracle.OK
            torch.cuda.synchronize(dst.device)
            assert p.audit() == 0
            assert_layers_equal([t.cpu().numpy() for t in dst.layers], expected)
        finally:
            p.close()
    finally:
        dst.close()
        src.close()
