"""§8 f3 groundwork: caches in exportable VMM memory (kvd_mem_alloc).

The prefill cache lives in a cuMemCreate allocation exported as a POSIX fd
(intra-node) or a fabric handle (multi-node NVLink, when IMEX permits it);
the decode side maps it and the unchanged pull kernel reads it.  Expected
bytes always come from the CPU oracle on regenerated seeded inputs.
"""
import multiprocessing as mp
import os
import sys

import numpy as np
import pytest
import torch

import kvdgen
from gpu_helpers import assert_layers_equal, make_pair, next_request_id, pull_and_wait
from paper_2501_14743_b200 import kvd

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = kvdgen.CacheGeom(4, 8, 128, 16, 256, kvdgen.BF16)


def test_mem_alloc_kinds_and_errors():
    ptr, size, kind = kvd.kvd_mem_alloc(0, 5 << 20)
    try:
        assert kind in (kvd.MEM_POSIX_FD, kvd.MEM_FABRIC)
        assert size >= 5 << 20 and size % (2 << 20) == 0 and ptr % (2 << 20) == 0
    finally:
        kvd.kvd_mem_free(ptr)
    with pytest.raises(kvd.KvdError) as ei:
        kvd.kvd_mem_free(ptr)                       # already freed
    assert ei.value.status == kvd.EINVAL
    with pytest.raises(kvd.KvdError) as ei:
        kvd.kvd_mem_alloc(0, 1 << 20, 5)            # unknown kind
    assert ei.value.status == kvd.EINVAL
    # FABRIC needs an IMEX channel: either granted or refused with EHANDLE
    try:
        ptr, _, kind = kvd.kvd_mem_alloc(0, 1 << 20, kvd.MEM_FABRIC)
        assert kind == kvd.MEM_FABRIC
        kvd.kvd_mem_free(ptr)
    except kvd.KvdError as e:
        assert e.status == kvd.EHANDLE, e


@pytest.mark.parametrize("src_mem,dst_mem", [("vmm", "vmm"), ("vmm", "torch"), ("torch", "vmm")])
def test_vmm_cache_pull_parity(src_mem, dst_mem):
    pair = make_pair(G, G, seed=90, src_memory=src_mem, dst_memory=dst_mem)
    try:
        tables = kvdgen.disjoint_fragmented_tables([100, 37, 64], 256, 256, seed=9)
        exp = pair.dst_host
        for s, d in tables:
            pull_and_wait(pair, s, d)
            exp = pair.expected(s, d, exp)
        assert_layers_equal(pair.download_dst(), exp)
    finally:
        pair.close()


def test_vmm_cache_pull_across_devices():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    pair = make_pair(G, G, seed=91, src_dev=0, dst_dev=1, src_memory="vmm", dst_memory="vmm")
    try:
        s, d = kvdgen.disjoint_fragmented_tables([200], 256, 256, seed=10)[0]
        pull_and_wait(pair, s, d)
        assert_layers_equal(pair.download_dst(), pair.expected(s, d))
    finally:
        pair.close()


def _prefill(conn, dev, released):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    torch.cuda.set_device(dev)
    from gpu_helpers import cache_for
    import kvdgen
    c = cache_for(G, dev, memory="vmm")
    for l in range(G.num_layers):
        c.layers[l].copy_(torch.from_numpy(kvdgen.random_bytes(c.layer_bytes, 700 + l)))
    torch.cuda.synchronize()
    conn.send((c.export(), c.mem_kind))
    conn.recv()          # decode finished and closed its peer
    released.put(sorted(c.poll_released()))
    c.close()


def _decode(conn, dev, result):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    torch.cuda.set_device(dev)
    from gpu_helpers import cache_for
    import kvdgen
    from oracle import oracle
    blob, kind = conn.recv()
    d = cache_for(G, dev)
    pre = [kvdgen.random_bytes(d.layer_bytes, 1900 + l) for l in range(G.num_layers)]
    for l in range(G.num_layers):
        d.layers[l].copy_(torch.from_numpy(pre[l]))
    torch.cuda.synchronize()
    peer = d.open_peer(blob)
    expected = [p.copy() for p in pre]
    src_host = [kvdgen.random_bytes(d.layer_bytes, 700 + l) for l in range(G.num_layers)]
    ok = True
    for k, (s, t) in enumerate(kvdgen.disjoint_fragmented_tables([100, 37, 64], 256, 256, 11)):
        peer.pull(8000 + k, s, t)
        peer.wait(8000 + k)
        rc = oracle.pull(src_host, G.stride, G.num_blocks, expected, G.stride, G.num_blocks,
                         G.num_kv_heads, G.head_dim, G.block_size, G.elem_bytes, s, t)
        ok = ok and rc == 0
    torch.cuda.synchronize()
    for l in range(G.num_layers):
        ok = ok and np.array_equal(d.layers[l].cpu().numpy(), expected[l])
    peer.close()
    d.close()
    conn.send("done")
    result.put((bool(ok), kind))


@pytest.mark.parametrize("devs", [(0, 0), (0, 1)])
def test_vmm_pull_across_processes(devs):
    """Exporter and importer in separate processes (one per GPU in
    deployment): the fd travels inside the blob and is fetched with
    pidfd_getfd; the release mailbox still reaches the exporter."""
    if max(devs) >= torch.cuda.device_count():
        pytest.skip("needs two GPUs")
    ctx = mp.get_context("spawn")
    a, b = ctx.Pipe()
    result, released = ctx.Queue(), ctx.Queue()
    p0 = ctx.Process(target=_prefill, args=(a, devs[0], released))
    p1 = ctx.Process(target=_decode, args=(b, devs[1], result))
    p0.start()
    p1.start()
    p1.join(300)
    p0.join(60)
    assert p1.exitcode == 0 and p0.exitcode == 0
    ok, kind = result.get(timeout=5)
    assert ok is True and kind in (kvd.MEM_POSIX_FD, kvd.MEM_FABRIC)
    assert released.get(timeout=5) == [8000, 8001, 8002]


def test_vmm_push_and_batch():
    """f2 push into an imported VMM decode cache, and an f1 batched drain from
    a VMM prefill cache: same oracle bytes as with cudaMalloc memory."""
    pair = make_pair(G, G, seed=92, src_memory="vmm", dst_memory="vmm")
    try:
        (s1, d1), (s2, d2), (s3, d3) = kvdgen.disjoint_fragmented_tables([50, 70, 30], 256, 256,
                                                                         seed=12)
        rev = pair.src.open_peer(pair.dst.export())   # prefill side imports the decode cache
        rid = next_request_id()
        rev.push(rid, s1, d1)
        rev.wait(rid)
        rev.close()
        exp = pair.expected(s1, d1)
        ids = [next_request_id(), next_request_id()]
        pair.peer.pull_batch(ids, [(s2, d2), (s3, d3)])
        for r in ids:
            pair.peer.wait(r)
        exp = pair.expected(s3, d3, pair.expected(s2, d2, exp))
        assert_layers_equal(pair.download_dst(), exp)
        assert sorted(pair.src.poll_released()) == sorted(ids)
    finally:
        pair.close()
