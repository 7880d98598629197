"""The N > 1 host path on CPU: world_size-2 (and 4, 8) gloo process groups run
the rail pairing, the one-time blob exchange (Connect()) and the
max-over-ranks aggregation that bench.py uses on the GPU box.  The blobs
are synthesised in the documented wire format and decoded by the C ABI's
host-only kvd_blob_info, so the codec is exercised across processes too.
"""
import os
import socket
import struct

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MAGIC = 0x4244564B


def make_blob(device, pid, layers=3, allocs=2, num_blocks=64, kinds=None, mailbox=False):
    """A blob in the wire format of kvd_export_handle, v4 (test-side encoder).
    kinds: per-allocation handle kind (0 legacy IPC, 1 POSIX fd, 8 fabric);
    mailbox: append the release-mailbox record (memfd number, bytes)."""
    kinds = kinds or [0] * allocs
    b = struct.pack("<IIII", MAGIC, 4, device, 0)
    b += struct.pack("<QQ", pid, 0xABCDEF)
    b += struct.pack("<IIIIII", layers, 2, 64, 16, num_blocks, 0)   # layers, heads, dim, bs, nb, fp16
    sub = 16 * 2 * 64
    b += struct.pack("<qqqqq", sub, num_blocks * sub, 128, 64, 1)
    b += struct.pack("<II", allocs, layers)
    layer_bytes = 2 * num_blocks * sub * 2
    for a in range(allocs):
        b += struct.pack("<II", kinds[a], 17 + a if kinds[a] == 1 else 0)
        b += bytes([a + 1]) * 64 + struct.pack("<QQ", 0x7F0000000000 + a * (1 << 32),
                                               layers * layer_bytes)
    for l in range(layers):
        b += struct.pack("<IIQ", l % allocs, 0, (l // allocs) * layer_bytes)
    if mailbox:
        b += struct.pack("<IIIQ", 1, 9, 0, 4 << 20)
    else:
        b += struct.pack("<I", 0)          # no release mailbox
    b += struct.pack("<I", MAGIC)
    return b


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_2501_14743_b200 import cluster, kvd
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        me = cluster.role_of(rank, world)
        mine = make_blob(rank, 1000 + rank) if me.role == "prefill" else None
        blobs = cluster.exchange_blobs(mine)
        got = cluster.peer_blob(me, blobs)
        res = {"rank": rank, "role": me.role, "peer": me.peer}
        if got is not None:
            layout, dev, pid, na = kvd.kvd_blob_info(got)
            res.update(blob_device=dev, blob_pid=pid, allocs=na, layers=layout.num_layers)
        # decode ranks "move" bytes; the job time is the max over them
        stats = {"bytes": (1 << 30) if me.role == "decode" else 0,
                 "dev_s": 0.001 * (rank + 1), "wall_s": 0.002 * (rank + 1)}
        res["agg"] = cluster.aggregate(cluster.gather_stats(stats))
        q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_pairing_exchange_and_aggregation_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted([q.get(timeout=10) for _ in range(world)], key=lambda r: r["rank"])
    half = world // 2
    for r in res:
        if r["rank"] < half:
            assert r["role"] == "prefill" and r["peer"] == r["rank"] + half
        else:
            # rail rule: decode rank half+k opened prefill rank k's blob
            assert r["role"] == "decode" and r["peer"] == r["rank"] - half
            assert r["blob_device"] == r["peer"] and r["blob_pid"] == 1000 + r["peer"]
            assert r["allocs"] == 2 and r["layers"] == 3
        agg = r["agg"]
        assert agg["ranks"] == half and agg["bytes"] == half * (1 << 30)
        assert agg["dev_s"] == pytest.approx(0.001 * world)      # max over decode ranks
        assert agg["wall_s"] == pytest.approx(0.002 * world)


def test_role_rules():
    from paper_2501_14743_b200 import cluster
    assert cluster.role_of(0, 1).role == "both"
    assert [cluster.role_of(r, 8).peer for r in range(8)] == [4, 5, 6, 7, 0, 1, 2, 3]
    with pytest.raises(ValueError):
        cluster.role_of(0, 3)
    with pytest.raises(ValueError):
        cluster.role_of(2, 2)


def test_synthesised_blob_round_trip_and_corruption():
    from paper_2501_14743_b200 import kvd
    blob = make_blob(5, 4242)
    layout, dev, pid, na = kvd.kvd_blob_info(blob)
    assert (dev, pid, na, layout.num_layers, layout.num_blocks) == (5, 4242, 2, 3, 64)
    assert list(layout.stride) == [2048, 64 * 2048, 128, 64, 1]
    for cut in (8, 40, len(blob) - 1):
        with pytest.raises(kvd.KvdError):
            kvd.kvd_blob_info(blob[:cut])
    bad = bytearray(blob)
    bad[-1] ^= 0xFF                                   # trailer
    with pytest.raises(kvd.KvdError):
        kvd.kvd_blob_info(bytes(bad))
    bad = bytearray(blob)
    off = len(blob) - 8 - 3 * 16                      # first layer's allocation index
    bad[off:off + 4] = struct.pack("<I", 7)
    with pytest.raises(kvd.KvdError):
        kvd.kvd_blob_info(bytes(bad))


def test_blob_handle_kinds():
    """The blob records a handle kind per allocation (legacy IPC, POSIX fd,
    fabric -- §8 f3 groundwork); unknown kinds and older versions are refused."""
    from paper_2501_14743_b200 import kvd
    for kinds in ([0, 0], [1, 1], [8, 0], [1, 8]):
        _, _, _, na = kvd.kvd_blob_info(make_blob(0, 1, kinds=kinds))
        assert na == 2
    with pytest.raises(kvd.KvdError) as ei:
        kvd.kvd_blob_info(make_blob(0, 1, kinds=[2, 0]))
    assert ei.value.status == kvd.EHANDLE
    old = bytearray(make_blob(0, 1))
    old[4:8] = struct.pack("<I", 2)
    with pytest.raises(kvd.KvdError):
        kvd.kvd_blob_info(bytes(old))


def test_blob_v4_mailbox_record():
    """Blob v4 carries the release mailbox as (memfd number, bytes) of the
    exporter's host memory; a truncated record, a bad flag or a v3 blob are
    refused."""
    from paper_2501_14743_b200 import kvd
    blob = make_blob(1, 77, mailbox=True)
    layout, dev, pid, na = kvd.kvd_blob_info(blob)
    assert (dev, pid, na) == (1, 77, 2)
    cut = blob[:-4 - 8] + blob[-4:]                   # mailbox record missing its size
    with pytest.raises(kvd.KvdError):
        kvd.kvd_blob_info(cut)
    bad = bytearray(blob)
    bad[-4 - 20:-4 - 16] = struct.pack("<I", 2)       # mailbox flag must be 0 or 1
    with pytest.raises(kvd.KvdError):
        kvd.kvd_blob_info(bytes(bad))
    v3 = bytearray(blob)
    v3[4:8] = struct.pack("<I", 3)
    with pytest.raises(kvd.KvdError):
        kvd.kvd_blob_info(bytes(v3))
