"""Cross-process pulls over CUDA IPC -- the deployment shape (one process per
GPU, P:L365-366 Connect(); "the decode worker reads the blocks from
the prefill worker").

A prefill process registers its caches and exports their blobs; a decode
process opens them (cudaIpcOpenMemHandle on cudaMalloc / torch memory, and
the exporter's release mailbox), pulls, polls, and compares its WHOLE
destination cache element by element with the CPU oracle run on host copies
of the same seeded inputs (regenerated in the decode process).  The prefill
process then reads the request ids that reached it one-sidedly through the
release mailbox.

Device pairs: (0, 0) runs on every box -- two processes on one GPU still go
through cudaIpcOpenMemHandle, the peer-mapped source address and the
cross-process mailbox, only the bytes stay in one HBM -- and (0, 1) over
NVLink when a second GPU exists.  Each pair runs every scenario in ONE
prefill/decode process pair (module-scoped fixture); each test asserts its
own scenario.  Besides the fixed scenarios, six seeded random serving
sequences (mover, resident engine, library streams, single pulls and
batches left in flight, kvd_poll_many) run across the processes too.
"""
import multiprocessing as mp
import os
import sys
import traceback

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

AUTO, LSU32, TMA = 0, 2, 4


def _small():
    import kvdgen
    return kvdgen.CacheGeom(4, 8, 128, 16, 256, kvdgen.BF16)


def _shard():   # a TP=8 prefill shard of the head-slice scenario (1 KV head)
    import kvdgen
    return kvdgen.CacheGeom(4, 1, 128, 16, 128, kvdgen.BF16)


def _exports():
    """name -> (geometry, single_allocation, content seed) of the prefill caches."""
    import kvdgen
    return {
        "small": (_small(), False, 500),
        "small_one_alloc": (_small(), True, 600),
        "c4": (kvdgen.C4, False, 700),
        "shard0": (_shard(), False, 800),
        "shard1": (_shard(), False, 900),
    }


# (name, source cache(s), mover, kind)
SCENARIOS = [
    ("tables_auto", "small", AUTO, "tables"),
    ("tables_one_alloc", "small_one_alloc", AUTO, "tables"),
    ("tables_tma", "small", TMA, "tables"),
    ("tables_lsu32", "small", LSU32, "tables"),
    ("c4_full_tma", "c4", TMA, "c4"),
    ("c4_full_lsu32", "c4", LSU32, "c4"),
    ("c4_full_auto", "c4", AUTO, "c4"),
    ("batch_auto", "small", AUTO, "batch"),
    ("batch_tma", "small", TMA, "batch"),
    ("batch_lsu32", "small", LSU32, "batch"),
    ("heads_auto", "shard0+shard1", AUTO, "heads"),
    ("heads_tma", "shard0+shard1", TMA, "heads"),
    ("engine_short", "small", AUTO, "engine"),
] + [(f"random{k}", "small", AUTO, f"random{k}") for k in range(6)]


def _paths():
    for p in (ROOT, os.path.join(ROOT, "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)


def _host(nbytes, seed, layers):
    import kvdgen
    return [kvdgen.random_bytes(nbytes, seed + l) for l in range(layers)]


def _prefill(conn, dev, released):
    _paths()
    import torch
    torch.cuda.set_device(dev)
    from gpu_helpers import cache_for
    caches = {}
    for name, (g, one, seed) in _exports().items():
        c = cache_for(g, dev, one)
        for l, h in enumerate(_host(c.layer_bytes, seed, g.num_layers)):
            c.layers[l].copy_(torch.from_numpy(h))
        caches[name] = c
    torch.cuda.synchronize()
    conn.send({name: c.export() for name, c in caches.items()})
    conn.recv()          # decode finished: only now may the exporter free its memory
    # Complete() reached this process one-sidedly through the release mailboxes
    released.put({name: sorted(c.poll_released()) for name, c in caches.items()})
    for c in caches.values():
        c.close()


def _scenario(kind, srcs, variant, blobs, dev, rid0):
    """Run one scenario in the decode process; returns the request ids it
    completed per source cache."""
    import torch
    import kvdgen
    from gpu_helpers import cache_for
    from oracle import oracle
    from paper_2501_14743_b200 import kvd
    ex = _exports()
    names = srcs.split("+")
    sg = ex[names[0]][0]
    if kind == "heads":
        dg = kvdgen.CacheGeom(sg.num_layers, 2 * sg.num_kv_heads, sg.head_dim, sg.block_size,
                              sg.num_blocks, sg.dtype)
    else:
        dg = sg
    d = cache_for(dg, dev)
    pre = _host(d.layer_bytes, 31 + rid0, dg.num_layers)
    for l in range(dg.num_layers):
        d.layers[l].copy_(torch.from_numpy(pre[l]))
    torch.cuda.synchronize()
    expected = pre
    done = {n: [] for n in names}
    rid = rid0
    if kind == "heads":
        peers = [d.open_peer_heads(blobs[n], i * sg.num_kv_heads) for i, n in enumerate(names)]
    else:
        peers = [d.open_peer(blobs[names[0]])]
    try:
        for p in peers:
            p.set(kvd.OPT_VARIANT, variant)
        from gpu_helpers import oracle_layer_bytes
        src_host = {n: _host(oracle_layer_bytes(sg), ex[n][2], sg.num_layers) for n in names}

        def oracle_pull(n, s, t, head_offset=None):
            if head_offset is None:
                rc = oracle.pull(src_host[n], sg.stride, sg.num_blocks, expected, dg.stride,
                                 dg.num_blocks, sg.num_kv_heads, sg.head_dim, sg.block_size,
                                 sg.elem_bytes, s, t)
            else:
                rc = oracle.pull_heads(src_host[n], sg.stride, sg.num_blocks, sg.num_kv_heads,
                                       expected, dg.stride, dg.num_blocks, dg.num_kv_heads,
                                       head_offset, sg.head_dim, sg.block_size, sg.elem_bytes,
                                       s, t)
            assert rc == oracle.OK, rc

        if kind.startswith("random"):           # a seeded serving sequence, requests in flight
            import random
            rng = random.Random(int(kind[6:]))
            p0 = peers[0]
            p0.set(kvd.OPT_VARIANT, rng.choice([AUTO, AUTO, TMA, LSU32]))
            p0.set(kvd.OPT_ENGINE, rng.choice([0, 8, 16]))
            p0.set(kvd.OPT_STREAMS, rng.choice([0, 0, 2]))
            sizes = [rng.choice([1, 2, 6, 20]) for _ in range(30)]
            while sum(sizes) > 180:             # ~70 % of the 256-block pool (room for gaps)
                sizes.pop()
            tables = kvdgen.disjoint_fragmented_tables(sizes, sg.num_blocks, dg.num_blocks,
                                                       100 + int(kind[6:]))
            pending, k = set(), 0
            while k < len(tables):
                if rng.random() < 0.2 and pending:
                    pending -= set(p0.poll_many(sorted(pending)))
                    continue
                m = rng.choice([1, 1, 1, 2, 3]) if k + 1 < len(tables) else 1
                m = min(m, len(tables) - k)
                ids = list(range(rid + 1, rid + 1 + m))
                rid += m
                if m == 1:
                    p0.pull(ids[0], *tables[k])
                else:
                    p0.pull_batch(ids, tables[k:k + m])
                for s, t in tables[k:k + m]:
                    oracle_pull(names[0], s, t)
                pending.update(ids)
                done[names[0]].extend(ids)
                k += m
            for r in sorted(pending):
                p0.wait(r)
        if kind == "engine":                    # short requests through the resident engine
            peers[0].set(kvd.OPT_ENGINE, 8)
            for s, t in kvdgen.disjoint_fragmented_tables([3, 7, 1, 5, 6] * 4, sg.num_blocks,
                                                          dg.num_blocks, 13):
                rid += 1
                peers[0].pull(rid, s, t)
                assert peers[0].info()["launches"] == 0
                peers[0].wait(rid)
                done[names[0]].append(rid)
                oracle_pull(names[0], s, t)
        if kind == "tables":
            for s, t in kvdgen.disjoint_fragmented_tables([100, 37, 64], sg.num_blocks,
                                                          dg.num_blocks, 8):
                rid += 1
                peers[0].pull(rid, s, t)
                peers[0].wait(rid)
                done[names[0]].append(rid)
                oracle_pull(names[0], s, t)
            info = peers[0].info()
            want = variant or (TMA if dev_pair_link[0] else LSU32)   # the auto policy
            assert info["variant"] == want, (info, want)
        elif kind == "c4":
            n = kvdgen.blocks_for(kvdgen.C4_TOKENS, sg.block_size)
            s, t = kvdgen.fragmented_table(n, sg.num_blocks, dg.num_blocks, seed=4)
            rid += 1
            peers[0].pull(rid, s, t)
            peers[0].wait(rid)
            done[names[0]].append(rid)
            info = peers[0].info()
            assert info["bytes"] == 671_088_640, info
            if variant:
                assert info["variant"] == variant, info
            oracle_pull(names[0], s, t)
        elif kind == "batch":
            tables = kvdgen.disjoint_fragmented_tables([40, 1, 0, 90, 33], sg.num_blocks,
                                                       dg.num_blocks, 11)
            # fig:queue shape: request 1 continues request 0's runs (merged across requests)
            ids = [rid + 1 + q for q in range(len(tables))]
            rid += len(tables)
            peers[0].pull_batch(ids, tables)
            for i in ids:
                peers[0].wait(i)
            done[names[0]].extend(ids)
            for s, t in tables:
                oracle_pull(names[0], s, t)
        elif kind == "heads":
            s, t = kvdgen.fragmented_table(70, sg.num_blocks, dg.num_blocks, seed=12)
            for i, (n, p) in enumerate(zip(names, peers)):
                rid += 1
                p.pull(rid, s, t)
                p.wait(rid)
                done[n].append(rid)
                oracle_pull(n, s, t, head_offset=i * sg.num_kv_heads)
        torch.cuda.synchronize()
        bad = []
        for l in range(dg.num_layers):
            got = d.layers[l].cpu().numpy()
            if not np.array_equal(got, expected[l]):
                k = np.flatnonzero(got != expected[l])
                bad.append(f"layer {l}: {k.size} bytes differ, first at {k[0]}")
        assert not bad, "; ".join(bad[:4])
    finally:
        for p in peers:
            p.close()
        d.close()
    return done


dev_pair_link = [False]


def _decode(conn, dev, link, result):
    _paths()
    import torch
    torch.cuda.set_device(dev)
    from paper_2501_14743_b200 import kvd
    dev_pair_link[0] = link
    blobs = conn.recv()
    out, released = {}, {}
    for name, blob in blobs.items():
        layout, _, pid, _ = kvd.kvd_blob_info(blob)
        assert pid != os.getpid()
    for k, (name, srcs, variant, kind) in enumerate(SCENARIOS):
        try:
            done = _scenario(kind, srcs, variant, blobs, dev, 10_000 * (k + 1))
            out[name] = "ok"
            for n, ids in done.items():
                released.setdefault(n, []).extend(ids)
        except Exception:
            out[name] = traceback.format_exc()[-3000:]
    conn.send("done")
    result.put((out, {n: sorted(v) for n, v in released.items()}))


_CACHE = {}


def _run_pair(devs):
    if devs in _CACHE:
        return _CACHE[devs]
    ctx = mp.get_context("spawn")
    a, b = ctx.Pipe()
    result, released = ctx.Queue(), ctx.Queue()
    p0 = ctx.Process(target=_prefill, args=(a, devs[0], released))
    p1 = ctx.Process(target=_decode, args=(b, devs[1], devs[0] != devs[1], result))
    p0.start()
    p1.start()
    try:
        out, want_released = result.get(timeout=900)
        got_released = released.get(timeout=120)
    finally:
        p1.join(60)
        p0.join(60)
        for p in (p0, p1):
            if p.is_alive():
                p.kill()
    _CACHE[devs] = (out, want_released, got_released, p0.exitcode, p1.exitcode)
    return _CACHE[devs]


DEVS = [(0, 0), (0, 1)]


def _need(devs):
    import torch
    if max(devs) >= torch.cuda.device_count():
        pytest.skip("needs two GPUs")


@pytest.mark.parametrize("devs", DEVS, ids=["same_gpu", "nvlink"])
@pytest.mark.parametrize("scenario", [s[0] for s in SCENARIOS])
def test_ipc_across_processes(devs, scenario):
    """Every scenario bit-exact against the oracle over a cross-process
    cudaIpcOpenMemHandle mapping (mover forced where named)."""
    _need(devs)
    out, _, _, _, _ = _run_pair(devs)
    assert out[scenario] == "ok", out[scenario]


@pytest.mark.parametrize("devs", DEVS, ids=["same_gpu", "nvlink"])
def test_ipc_release_ids_reach_prefill(devs):
    """Complete() -> prefill: every request the decode
    process completed is reported exactly once by kvd_poll_released in the
    exporting process, per exported cache; both processes exit cleanly."""
    _need(devs)
    out, want, got, rc0, rc1 = _run_pair(devs)
    assert rc0 == 0 and rc1 == 0
    for name in _exports():
        assert got.get(name, []) == want.get(name, []), name
