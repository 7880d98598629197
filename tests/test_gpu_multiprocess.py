"""Cross-process pull over CUDA IPC (the real deployment shape: one process
per GPU).  The prefill process registers + exports; the decode process opens
the blob (cudaIpcOpenMemHandle -> NVLink mapping), pulls, polls and checks
the result against the oracle on regenerated seeded inputs.
"""
import multiprocessing as mp
import os
import sys

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.gpu2]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _geom():
    import kvdgen
    return kvdgen.CacheGeom(4, 8, 128, 16, 256, kvdgen.BF16)


def _prefill(conn, dev, single_alloc, released):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    torch.cuda.set_device(dev)
    from gpu_helpers import cache_for
    import kvdgen
    g = _geom()
    c = cache_for(g, dev, single_alloc)
    for l in range(g.num_layers):
        c.layers[l].copy_(torch.from_numpy(kvdgen.random_bytes(c.layer_bytes, 500 + l)))
    torch.cuda.synchronize()
    conn.send(c.export())
    conn.recv()          # decode finished: now the exporter may free its memory
    # Complete() reached this process one-sidedly through the release mailbox
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
    from paper_2501_14743_b200 import kvd
    g = _geom()
    blob = conn.recv()
    layout, exp_dev, pid, nalloc = kvd.kvd_blob_info(blob)
    assert pid != os.getpid() and layout.num_layers == g.num_layers
    d = cache_for(g, dev)
    pre = [kvdgen.random_bytes(d.layer_bytes, 900 + l) for l in range(g.num_layers)]
    for l in range(g.num_layers):
        d.layers[l].copy_(torch.from_numpy(pre[l]))
    torch.cuda.synchronize()
    peer = d.open_peer(blob)
    ok = True
    expected = [p.copy() for p in pre]
    src_host = [kvdgen.random_bytes(d.layer_bytes, 500 + l) for l in range(g.num_layers)]
    for k, (s, t) in enumerate(kvdgen.disjoint_fragmented_tables([100, 37, 64], 256, 256, 8)):
        peer.pull(7000 + k, s, t)
        peer.wait(7000 + k)
        rc = oracle.pull(src_host, g.stride, g.num_blocks, expected, g.stride, g.num_blocks,
                         g.num_kv_heads, g.head_dim, g.block_size, g.elem_bytes, s, t)
        ok = ok and rc == 0
    torch.cuda.synchronize()
    for l in range(g.num_layers):
        ok = ok and np.array_equal(d.layers[l].cpu().numpy(), expected[l])
    peer.close()
    d.close()
    conn.send("done")
    result.put(bool(ok))


@pytest.mark.parametrize("single_alloc", [False, True])
def test_ipc_pull_across_processes(single_alloc):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    ctx = mp.get_context("spawn")
    a, b = ctx.Pipe()
    result = ctx.Queue()
    released = ctx.Queue()
    p0 = ctx.Process(target=_prefill, args=(a, 0, single_alloc, released))
    p1 = ctx.Process(target=_decode, args=(b, 1, result))
    p0.start()
    p1.start()
    p1.join(300)
    p0.join(60)
    assert p1.exitcode == 0 and p0.exitcode == 0
    assert result.get(timeout=5) is True
    assert released.get(timeout=5) == [7000, 7001, 7002]
