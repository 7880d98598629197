"""§8 f1 -- batched drain: several requests in ONE launch, runs coalesced
across requests (fig:queue), each request completed on its own.
Expected bytes always come from the oracle applying the requests in order
(destinations are disjoint, so any order gives the same bytes)."""
import numpy as np
import pytest
import torch

import kvdgen
from gpu_helpers import assert_layers_equal, make_pair, next_request_id
from paper_2501_14743_b200 import kvd

pytestmark = pytest.mark.gpu

G = kvdgen.CacheGeom(2, 2, 64, 16, 512, kvdgen.FP16)


def _expected(pair, tables):
    exp = pair.dst_host
    for s, d in tables:
        exp = pair.expected(s, d, exp)
    return exp


def _run_batch(pair, tables):
    rids = [next_request_id() for _ in tables]
    pair.peer.pull_batch(rids, tables)
    for rid in reversed(rids):
        pair.peer.wait(rid)
    return rids


@pytest.mark.parametrize("variant", [kvd.VARIANT_AUTO, kvd.VARIANT_LSU, kvd.VARIANT_TMA])
@pytest.mark.parametrize("counts", [[16], [16, 5, 30, 1, 9, 40], [0, 7, 0, 3], [64] * 8])
def test_batch_bit_exact(variant, counts):
    pair = make_pair(G, G, seed=30)
    try:
        pair.peer.set(kvd.OPT_VARIANT, variant)
        if variant == kvd.VARIANT_TMA:
            pair.peer.set(kvd.OPT_TILE_BYTES, 4096)
        tables = kvdgen.disjoint_fragmented_tables(counts, 512, 512, seed=sum(counts))
        _run_batch(pair, tables)
        assert_layers_equal(pair.download_dst(), _expected(pair, tables))
    finally:
        pair.close()


def test_batch_merges_across_requests_fig_queue():
    """R1 reads remote 0 -> local 5, R2 reads remote 1 -> local 6: one run."""
    pair = make_pair(G, G, seed=31)
    try:
        tables = [(np.array([0], np.int32), np.array([5], np.int32)),
                  (np.array([1], np.int32), np.array([6], np.int32))]
        _run_batch(pair, tables)
        assert pair.peer.info()["runs"] == 1
        assert_layers_equal(pair.download_dst(), _expected(pair, tables))
        # runs spanning many requests whose blocks share tiles (span 4 KiB,
        # tile 16 KiB): every request still completes exactly once
        pair.peer.set(kvd.OPT_TILE_BYTES, 16384)
        base = 100
        tables = [(np.arange(base + 3 * i, base + 3 * i + 3, dtype=np.int32),
                   np.arange(300 + 3 * i, 300 + 3 * i + 3, dtype=np.int32)) for i in range(20)]
        pre = pair.download_dst()
        _run_batch(pair, tables)
        assert pair.peer.info()["runs"] == 1
        exp = pre
        for s, d in tables:
            exp = pair.expected(s, d, exp)
        assert_layers_equal(pair.download_dst(), exp)
    finally:
        pair.close()


def test_batch_errors():
    pair = make_pair(G, G, seed=32)
    try:
        a = (np.array([1, 2], np.int32), np.array([3, 4], np.int32))
        b = (np.array([5], np.int32), np.array([4], np.int32))       # dst 4 twice
        with pytest.raises(kvd.KvdError) as ei:
            pair.peer.pull_batch([next_request_id(), next_request_id()], [a, b])
        assert ei.value.status == kvd.EINVAL
        rid = next_request_id()
        with pytest.raises(kvd.KvdError) as ei:
            pair.peer.pull_batch([rid, rid], [a, (b[0], np.array([9], np.int32))])
        assert ei.value.status == kvd.EINVAL
        torch.cuda.synchronize()
        assert_layers_equal(pair.download_dst(), pair.dst_host)
    finally:
        pair.close()


def test_batch_per_request_completion_and_reuse():
    """Many batches back to back; descriptor buffers are recycled only after
    every request of a batch retired; data never precedes its flag."""
    pair = make_pair(G, G, seed=33)
    rng = np.random.default_rng(3)
    span = pair.src.span_bytes
    src_view = [torch.from_numpy(h).view(2, 512, span) for h in pair.src_host]
    side = torch.cuda.Stream()
    try:
        for it in range(300):
            counts = [int(c) for c in rng.integers(0, 12, size=int(rng.integers(1, 6)))]
            tables = kvdgen.disjoint_fragmented_tables(counts, 512, 512, seed=it)
            rids = [next_request_id() for _ in tables]
            pair.peer.pull_batch(rids, tables)
            for rid, (s, d) in zip(rids, tables):
                while not pair.peer.poll(rid):
                    pass
                if len(d) == 0:
                    continue
                with torch.cuda.stream(side):
                    got = [t.view(2, 512, span)[:, torch.from_numpy(d).long().cuda()].cpu()
                           for t in pair.dst.layers]
                for l in range(G.num_layers):
                    assert torch.equal(got[l], src_view[l][:, torch.from_numpy(s).long()])
    finally:
        pair.close()


@pytest.mark.gpu2
def test_batch_two_gpus_c2_shaped():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    g = kvdgen.CacheGeom(8, 32, 128, 16, 1024, kvdgen.FP16)
    pair = make_pair(g, g, seed=34, src_dev=0, dst_dev=1)
    try:
        toks = kvdgen.mixed_request_tokens(8, seed=2, lo=256, hi=1536)
        counts = [kvdgen.blocks_for(t, 16) for t in toks]
        tables = kvdgen.disjoint_fragmented_tables(counts, 1024, 1024, seed=5)
        _run_batch(pair, tables)
        assert_layers_equal(pair.download_dst(), _expected(pair, tables))
    finally:
        pair.close()
