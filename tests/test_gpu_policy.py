"""The auto launch policy: which mover and grid a request gets,
checked through kvd_last_pull_info, each case also bit-exact against the
oracle.  Small requests (<= 2 MiB) -> one-warp CTAs and 2 KiB tiles; medium
loopback requests -> at least two CTAs per SM; over NVLink -> the TMA ring
with >= 48 CTAs."""
import pytest
import torch

import kvdgen
from gpu_helpers import assert_layers_equal, make_pair, pull_and_wait

pytestmark = pytest.mark.gpu

G7B = kvdgen.C2.with_blocks(48)      # Llama-2-7B geometry, 8 MiB per block, small pools


def _sms(dev=0):
    return torch.cuda.get_device_properties(dev).multi_processor_count


def test_small_request_policy():
    g = kvdgen.C1
    pair = make_pair(g, g, seed=101)
    try:
        s, d = kvdgen.fragmented_table(16, g.num_blocks, g.num_blocks, seed=3)
        info = pull_and_wait(pair, s, d)
        assert info["threads"] == 32 and info["variant"] == 2   # LSU32, one warp per CTA
        assert info["tiles"] == info["ctas"]                     # one 2 KiB tile per warp
        assert_layers_equal(pair.download_dst(), pair.expected(s, d))
    finally:
        pair.close()


@pytest.mark.parametrize("blocks", [1, 2, 4, 16])
def test_medium_loopback_request_spreads_over_the_gpu(blocks):
    pair = make_pair(G7B, G7B, seed=102)
    try:
        s, d = kvdgen.fragmented_table(blocks, G7B.num_blocks, G7B.num_blocks, seed=blocks)
        info = pull_and_wait(pair, s, d)
        assert info["variant"] == 2
        assert info["ctas"] >= min(2 * _sms(), info["tiles"]), info
        assert_layers_equal(pair.download_dst(), pair.expected(s, d))
    finally:
        pair.close()


def test_large_loopback_request_uses_full_chunks():
    pair = make_pair(G7B, G7B, seed=103)
    try:
        s, d = kvdgen.fragmented_table(40, G7B.num_blocks, G7B.num_blocks, seed=4)
        info = pull_and_wait(pair, s, d)
        assert info["variant"] == 2 and info["threads"] == 512
        assert_layers_equal(pair.download_dst(), pair.expected(s, d))
    finally:
        pair.close()


def test_over_nvlink_uses_tma_ring():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    pair = make_pair(G7B, G7B, seed=104, src_dev=0, dst_dev=1)
    try:
        s, d = kvdgen.fragmented_table(32, G7B.num_blocks, G7B.num_blocks, seed=5)
        info = pull_and_wait(pair, s, d)
        assert info["variant"] == 4 and info["ctas"] >= 48
        assert_layers_equal(pair.download_dst(), pair.expected(s, d))
    finally:
        pair.close()


def test_short_nvlink_requests_get_more_ctas():
    """<= 48 MiB over NVLink: at least 96 CTAs (the request is in flight almost
    whole from the first ring); longer requests keep the 48-CTA floor."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    g = kvdgen.C4.with_blocks(256)
    pair = make_pair(g, g, seed=108, src_dev=0, dst_dev=1)
    try:
        exp = pair.dst_host
        for blocks, lo, hi in ((8, 96, 148), (128, 48, 95)):
            s, d = kvdgen.fragmented_table(blocks, g.num_blocks, g.num_blocks, seed=blocks)
            info = pull_and_wait(pair, s, d)
            assert info["variant"] == 4 and lo <= info["ctas"] <= hi, (blocks, info)
            exp = pair.expected(s, d, exp)          # the second pull lands on the first's result
            assert_layers_equal(pair.download_dst(), exp)
    finally:
        pair.close()


def test_device_time_globaltimer_cross_check():
    """KVD_OPT_TIMING: the in-kernel %globaltimer span (first CTA start ->
    last CTA done) of each retired single pull, next to the CUDA-event time
    around the launch (which also holds the launch latency)."""
    from paper_2501_14743_b200 import kvd
    pair = make_pair(G7B, G7B, seed=105)
    try:
        pair.peer.set(kvd.OPT_TIMING, 1)
        s, d = kvdgen.fragmented_table(32, G7B.num_blocks, G7B.num_blocks, seed=6)
        for _ in range(3):
            pull_and_wait(pair, s, d)
        gt_ms, n = pair.peer.device_time()
        ev_ms, m = pair.peer.kernel_time()
        assert n == 3 and m == 3
        assert 0 < gt_ms <= ev_ms * 1.02, (gt_ms, ev_ms)
        # 256 MiB each way through one HBM: no faster than ~10 TB/s of r+w
        assert gt_ms / 3 > 2 * 32 * G7B.num_layers * 2 * (128 << 10) / 10e12 * 1e3
        assert pair.peer.device_time() == (0.0, 0)              # reset by the read
        pair.peer.set(kvd.OPT_TIMING, 0)
        pull_and_wait(pair, s, d)
        assert pair.peer.device_time() == (0.0, 0)              # off: nothing recorded
        assert_layers_equal(pair.download_dst(), pair.expected(s, d))
    finally:
        pair.close()


def test_link_calibration_reads_only():
    """kvd_peer_calibrate (SURVEY §8 d, the measured link ceiling): pure bulk
    reads of the source layers.  Loopback reads local HBM (no write traffic,
    so above the HBM copy rate's read half); errors on bad sizes; and it
    leaves both caches untouched."""
    from paper_2501_14743_b200 import kvd
    pair = make_pair(G7B, G7B, seed=106)
    try:
        before_src = [t.clone() for t in pair.src.layers]
        before_dst = [t.clone() for t in pair.dst.layers]
        total = G7B.num_layers * pair.src.layer_bytes
        gbs = pair.peer.calibrate(min(total, 1 << 30), reps=2)
        assert 1000 < gbs < 9000, gbs
        with pytest.raises(kvd.KvdError) as e:
            pair.peer.calibrate(1024)
        assert e.value.status == kvd.EINVAL
        with pytest.raises(kvd.KvdError) as e:
            pair.peer.calibrate(total + (1 << 20))
        assert e.value.status == kvd.ERANGE
        with pytest.raises(kvd.KvdError) as e:
            pair.peer.calibrate(1 << 20, stages=8)
        assert e.value.status == kvd.EINVAL
        torch.cuda.synchronize()
        for a, b in zip(before_src, pair.src.layers):
            assert torch.equal(a, b)
        for a, b in zip(before_dst, pair.dst.layers):
            assert torch.equal(a, b)
    finally:
        pair.close()


def test_link_calibration_over_nvlink():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    pair = make_pair(G7B, G7B, seed=107, src_dev=0, dst_dev=1)
    try:
        total = G7B.num_layers * (pair.src.layer_bytes // 32768) * 32768
        gbs = max(pair.peer.calibrate(total, ctas=c, reps=2) for c in (48, 148))
        assert 600 < gbs < 900, gbs      # NVLink 5: 900 GB/s per direction on the wire
    finally:
        pair.close()


@pytest.mark.parametrize("opts", [{"threads": 512}, {"threads": 256, "tile": 65536},
                                  {"tile": 131072}, {"threads": 512, "tile": 131072,
                                                     "stages": 3}])
def test_auto_over_nvlink_fits_caller_options(opts):
    """AUTO picks the TMA ring over NVLink; options a caller set with the LSU
    mover in mind (512 threads, big tiles) are fitted to the ring's shared
    memory -- fewer pipes or stages, or the LSU mover when one pipe's ring
    cannot hold two tiles -- instead of failing (a fuzz case did)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    from paper_2501_14743_b200 import kvd
    pair = make_pair(G7B, G7B, seed=109, src_dev=0, dst_dev=1)
    try:
        names = {"threads": kvd.OPT_THREADS, "tile": kvd.OPT_TILE_BYTES, "stages": kvd.OPT_STAGES}
        for k, v in opts.items():
            pair.peer.set(names[k], v)
        s, d = kvdgen.fragmented_table(24, G7B.num_blocks, G7B.num_blocks, seed=9)
        info = pull_and_wait(pair, s, d)
        if info["variant"] == 4:
            assert info["threads"] <= 256
        assert_layers_equal(pair.download_dst(), pair.expected(s, d))
    finally:
        pair.close()
