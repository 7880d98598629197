"""The resident pull engine (KVD_OPT_ENGINE): short requests are posted as
descriptors into a pinned ring that a persistent kernel drains (the paper's
transaction queue, posted straight to the device).  Every result
is compared with the CPU oracle; completion must never precede the data
(SURVEY §8 c P4); the engine exits when idle and restarts on demand."""
import time

import numpy as np
import pytest
import torch

import kvdgen
from gpu_helpers import assert_layers_equal, make_pair, next_request_id
from paper_2501_14743_b200 import kvd

pytestmark = pytest.mark.gpu

G = kvdgen.CacheGeom(2, 2, 64, 16, 256, kvdgen.FP16)     # 4 KiB spans


def _engine_pair(seed, ctas=8, g=G):
    pair = make_pair(g, g, seed=seed)
    pair.peer.set(kvd.OPT_ENGINE, ctas)
    return pair


@pytest.mark.parametrize("ctas", [1, 3, 8, 16])
def test_engine_small_pulls_bit_exact(ctas):
    pair = _engine_pair(90 + ctas, ctas)
    try:
        with pytest.raises(kvd.KvdError):
            pair.peer.set(kvd.OPT_ENGINE, 17)             # one cluster: at most 16 CTAs
        rng = np.random.default_rng(ctas)
        exp = pair.dst_host
        for it in range(60):
            n = int(rng.integers(1, 64))
            s = rng.choice(256, n, replace=False).astype(np.int32)
            d = rng.choice(256, n, replace=False).astype(np.int32)
            rid = next_request_id()
            pair.peer.pull(rid, s, d)
            info = pair.peer.info()
            assert info["launches"] == 0 and info["ctas"] == ctas, info   # posted, not launched
            pair.peer.wait(rid)
            exp = pair.expected(s, d, exp)
        assert_layers_equal(pair.download_dst(), exp)
    finally:
        pair.close()


def test_engine_many_in_flight_then_poll():
    """Hundreds of requests posted back to back (more than the 128-entry
    ring: the overflow takes the launch path) with disjoint destinations."""
    g = kvdgen.CacheGeom(2, 2, 64, 16, 4096, kvdgen.FP16)
    pair = _engine_pair(95, 8, g)
    try:
        tables = kvdgen.disjoint_fragmented_tables([6] * 300, 4096, 4096, seed=5)
        rids, launched = [], 0
        for s, d in tables:
            rid = next_request_id()
            pair.peer.pull(rid, s, d)
            launched += pair.peer.info()["launches"]
            rids.append(rid)
        pending = list(rids)
        while pending:
            done = pair.peer.poll_many(pending)
            pending = [r for r in pending if r not in done]
        exp = pair.dst_host
        for s, d in tables:
            exp = pair.expected(s, d, exp)
        assert_layers_equal(pair.download_dst(), exp)
        assert sorted(pair.src.poll_released()) == sorted(rids)
        print(f"{launched} of {len(rids)} requests took the launch path")
    finally:
        pair.close()


def test_engine_completion_never_precedes_data():
    """P4 with the engine: the first time kvd_poll_done returns 1 the host
    reads the destination blocks on another stream; they hold the bytes."""
    pair = _engine_pair(96)
    side = torch.cuda.Stream()
    rng = np.random.default_rng(1)
    span = pair.src.span_bytes
    try:
        src_view = [torch.from_numpy(h).view(2, 256, span) for h in pair.src_host]
        for it in range(1500):
            n = int(rng.integers(1, 65))
            s = rng.choice(256, n, replace=False).astype(np.int32)
            d = rng.choice(256, n, replace=False).astype(np.int32)
            rid = next_request_id()
            pair.peer.pull(rid, s, d)
            while not pair.peer.poll(rid):
                pass
            with torch.cuda.stream(side):
                got = [t.view(2, 256, span)[:, torch.from_numpy(d).long().cuda()].cpu()
                       for t in pair.dst.layers]
            for l in range(G.num_layers):
                want = src_view[l][:, torch.from_numpy(s).long()]
                assert torch.equal(got[l], want), f"iteration {it} layer {l}: flag before data"
    finally:
        pair.close()


def test_engine_and_launch_path_mixed():
    """A request above 2 MiB (or a forced variant) takes the launch path
    while the engine serves the short ones; every byte is the oracle's."""
    g = kvdgen.CacheGeom(4, 8, 128, 16, 512, kvdgen.FP16)   # 32 KiB spans: 8 blocks = 2 MiB
    pair = _engine_pair(97, 8, g)
    try:
        tables = kvdgen.disjoint_fragmented_tables([3, 40, 5, 100, 2], 512, 512, seed=6)
        paths = []
        for s, d in tables:
            rid = next_request_id()
            pair.peer.pull(rid, s, d)
            paths.append(pair.peer.info()["launches"])
            pair.peer.wait(rid)
        assert paths == [0, 1, 0, 1, 0], paths
        exp = pair.dst_host
        for s, d in tables:
            exp = pair.expected(s, d, exp)
        assert_layers_equal(pair.download_dst(), exp)
    finally:
        pair.close()


def test_engine_idle_exit_restart_and_stop():
    """Idle for longer than the 2 ms timeout the engine exits (a device-wide
    synchronise returns); the next short request relaunches it; turning it
    off mid-stream completes what was posted."""
    pair = _engine_pair(98)
    try:
        exp = pair.dst_host
        for rep in range(3):
            s, d = kvdgen.random_table(10, 256, 256, seed=rep)
            rid = next_request_id()
            pair.peer.pull(rid, s, d)
            pair.peer.wait(rid)
            exp = pair.expected(s, d, exp)
            time.sleep(0.02)
            t0 = time.perf_counter()
            torch.cuda.synchronize()
            assert time.perf_counter() - t0 < 1.0
        rids = []
        for k in range(20):
            s, _ = kvdgen.random_table(5, 256, 256, seed=100 + k)
            rid = next_request_id()
            d = np.arange(5 * k, 5 * k + 5, dtype=np.int32)
            pair.peer.pull(rid, s, d)
            exp = pair.expected(s, d, exp)
            rids.append(rid)
        pair.peer.set(kvd.OPT_ENGINE, 0)                  # posted requests still complete
        for r in rids:
            pair.peer.wait(r)
        assert_layers_equal(pair.download_dst(), exp)
        s, d = kvdgen.random_table(7, 256, 256, seed=7)
        rid = next_request_id()
        pair.peer.pull(rid, s, d)                          # engine off: launch path
        assert pair.peer.info()["launches"] == 1
        pair.peer.wait(rid)
    finally:
        pair.close()


def test_engine_close_while_live():
    pair = _engine_pair(99)
    try:
        s, d = kvdgen.random_table(12, 256, 256, seed=3)
        rid = next_request_id()
        pair.peer.pull(rid, s, d)
        pair.peer.wait(rid)
    finally:
        pair.close()                                       # stops the live engine first
    torch.cuda.synchronize()


@pytest.mark.timeout(300, method="thread")
def test_engine_live_during_device_synchronising_calls():
    """Calls that synchronise the device under the peer mutex -- the first
    batched drain (descriptor buffer allocation) and a > 2016-run table
    outgrowing its slot's device buffer (cudaFree) -- made while the engine
    is live must stop it first (its idle watchdog cannot take the mutex):
    before the fix this sequence deadlocked (a 800-seed fuzz soak hung)."""
    g = kvdgen.CacheGeom(2, 2, 64, 16, 8192, kvdgen.FP16)   # 4 KiB spans
    pair = _engine_pair(97, 16, g)
    try:
        exp = pair.dst_host

        def short():                              # posted to the engine, leaves it live
            s, d = kvdgen.fragmented_table(8, 8192, 8192, seed=next_request_id() % 1000)
            rid = next_request_id()
            pair.peer.pull(rid, s, d)
            assert pair.peer.info()["launches"] == 0
            pair.peer.wait(rid)
            return s, d

        s, d = short()
        exp = pair.expected(s, d, exp)
        tables = kvdgen.disjoint_fragmented_tables([40, 24], 8192, 8192, seed=7)
        rids = [next_request_id() for _ in tables]
        pair.peer.pull_batch(rids, tables)       # first batch: allocates its buffer
        for r in rids:
            pair.peer.wait(r)
        for s_, d_ in tables:
            exp = pair.expected(s_, d_, exp)
        rid = next_request_id()
        for n in (2100, 2300):                   # the same id -> the same slot, a bigger table
            s, d = short()
            exp = pair.expected(s, d, exp)
            src = np.arange(0, 2 * n, 2, dtype=np.int32)          # every other block: n runs
            dst = np.arange(1, 2 * n + 1, 2, dtype=np.int32)[::-1].copy()
            pair.peer.pull(rid, src, dst)
            assert pair.peer.info()["runs"] == n
            pair.peer.wait(rid)
            exp = pair.expected(src, dst, exp)
        assert_layers_equal(pair.download_dst(), exp)
    finally:
        pair.close()
