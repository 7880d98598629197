"""GPU parity of the pull path (C ABI -> sm_100a kernel) against the CPU oracle.

Every test compares the decode cache after kvd_pull, byte for byte, with the
oracle's result on host copies of the same seeded inputs (SURVEY.md §8 row c
P3: unique result, bit-exact).  On a one-GPU box the prefill and decode
caches share the GPU (loopback); tests marked gpu2 use two GPUs.
"""
import numpy as np
import pytest
import torch

import kvdgen
from gpu_helpers import (assert_layers_equal, make_pair, next_request_id, pull_and_wait)
from paper_2501_14743_b200 import kvd

pytestmark = pytest.mark.gpu

C1 = kvdgen.C1
N_C1 = kvdgen.blocks_for(kvdgen.C1_TOKENS, C1.block_size)


def _tables(kind, n, nb_s, nb_d, seed):
    if kind == "contiguous":
        return kvdgen.contiguous_table(n, 0, nb_d - n)
    if kind == "fragmented":
        return kvdgen.fragmented_table(n, nb_s, nb_d, seed)
    if kind == "random":
        return kvdgen.random_table(n, nb_s, nb_d, seed)
    if kind == "reversed":
        s, d = kvdgen.contiguous_table(n, 0, 0)
        return s, d[::-1].copy()
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["contiguous", "fragmented", "random", "reversed"])
def test_c1_bit_exact(kind):
    pair = make_pair(C1, C1, seed=1)
    try:
        src, dst = _tables(kind, N_C1, C1.num_blocks, C1.num_blocks, seed=0)
        info = pull_and_wait(pair, src, dst)
        assert info["blocks"] == N_C1 and info["bytes"] == N_C1 * C1.num_layers * 2 * 4096
        assert_layers_equal(pair.download_dst(), pair.expected(src, dst))
        # I3: the source cache is unchanged
        torch.cuda.synchronize()
        for l, t in enumerate(pair.src.layers):
            assert np.array_equal(t.cpu().numpy(), pair.src_host[l])
    finally:
        pair.close()


SUB = 16 * 2 * 64   # C1 sub-tensor elements


@pytest.mark.parametrize("sstride,dstride", [
    ((0,) * 5, (0,) * 5),                                                  # Fig. 5 / vLLM flash
    ((2 * SUB, SUB, 128, 64, 1), (2 * SUB, SUB, 128, 64, 1)),              # block-major: K,V fold
    ((3 * SUB, SUB, 128, 64, 1), (2 * SUB + 64, SUB, 128, 64, 1)),         # padded: non-contiguous
    ((0,) * 5, (2 * SUB, SUB, 128, 64, 1)),                                # mixed orders
    ((SUB + 128, 64 * (SUB + 128), 128, 64, 1), (0,) * 5),                 # padded KV-outer
])
def test_layouts_bit_exact(sstride, dstride):
    sg = kvdgen.CacheGeom(2, 2, 64, 16, 64, kvdgen.FP16, sstride)
    dg = kvdgen.CacheGeom(2, 2, 64, 16, 64, kvdgen.FP16, dstride)
    pair = make_pair(sg, dg, seed=2)
    try:
        for kind in ("fragmented", "random", "contiguous"):
            src, dst = _tables(kind, 20, 64, 64, seed=5)
            pre = pair.download_dst()
            pull_and_wait(pair, src, dst)
            assert_layers_equal(pair.download_dst(), pair.expected(src, dst, pre))
    finally:
        pair.close()


@pytest.mark.parametrize("geom", [
    kvdgen.CacheGeom(3, 1, 16, 8, 50, kvdgen.FP8),         # 128 B spans
    kvdgen.CacheGeom(2, 4, 128, 32, 40, kvdgen.FP32),      # 64 KiB spans: several tiles per block
    kvdgen.CacheGeom(80, 2, 128, 16, 64, kvdgen.BF16),     # C4 shard geometry, small pool
    kvdgen.CacheGeom(1, 1, 8, 1, 300, kvdgen.FP16),        # 16 B spans (minimum)
])
def test_geometries_bit_exact(geom):
    pair = make_pair(geom, geom.with_blocks(geom.num_blocks + 7), seed=3)
    try:
        n = min(geom.num_blocks, 37)
        src, dst = kvdgen.fragmented_table(n, geom.num_blocks, geom.num_blocks + 7, seed=9)
        pull_and_wait(pair, src, dst)
        assert_layers_equal(pair.download_dst(), pair.expected(src, dst))
    finally:
        pair.close()


@pytest.mark.parametrize("variant", [kvd.VARIANT_LSU, kvd.VARIANT_LSU32, kvd.VARIANT_CE,
                                     kvd.VARIANT_TMA])
@pytest.mark.parametrize("tile", [512, 4096, 16384, 65536])
def test_variants_and_tiles(variant, tile):
    g = kvdgen.CacheGeom(4, 4, 64, 16, 96, kvdgen.FP16)   # 8 KiB spans
    pair = make_pair(g, g, seed=4)
    try:
        pair.peer.set(kvd.OPT_VARIANT, variant).set(kvd.OPT_TILE_BYTES, tile)
        if variant == kvd.VARIANT_TMA and tile == 65536:
            pair.peer.set(kvd.OPT_THREADS, 32).set(kvd.OPT_STAGES, 3)   # fit 227 KiB
        src, dst = kvdgen.fragmented_table(60, 96, 96, seed=tile)
        info = pull_and_wait(pair, src, dst)
        assert info["variant"] == variant
        assert_layers_equal(pair.download_dst(), pair.expected(src, dst))
    finally:
        pair.close()


@pytest.mark.parametrize("threads,max_ctas", [(128, 1), (512, 3), (512, 0), (256, 7), (32, 0)])
def test_grid_shapes(threads, max_ctas):
    pair = make_pair(C1, C1, seed=5)
    try:
        pair.peer.set(kvd.OPT_THREADS, threads).set(kvd.OPT_MAX_CTAS, max_ctas)
        src, dst = kvdgen.random_table(N_C1, 64, 64, seed=2)
        info = pull_and_wait(pair, src, dst)
        if max_ctas:
            assert info["ctas"] <= max_ctas
        assert_layers_equal(pair.download_dst(), pair.expected(src, dst))
    finally:
        pair.close()


def test_coalesce_off_same_bytes():
    """E10 ablation switch: coalescing changes the descriptor count, never the bytes."""
    pair = make_pair(C1, C1, seed=6)
    try:
        src, dst = kvdgen.contiguous_table(N_C1, 3, 40)
        info_on = pull_and_wait(pair, src, dst)
        assert info_on["runs"] == 1
        pair.upload_dst(pair.dst_host)
        pair.peer.set(kvd.OPT_COALESCE, 0)
        info_off = pull_and_wait(pair, src, dst)
        assert info_off["runs"] == N_C1
        assert_layers_equal(pair.download_dst(), pair.expected(src, dst))
    finally:
        pair.close()


def test_run_table_in_device_memory():
    """More runs than fit in kernel parameters (> 2016): the per-slot device
    run table path."""
    g = kvdgen.CacheGeom(2, 1, 8, 1, 6000, kvdgen.FP16)
    pair = make_pair(g, g, seed=7)
    try:
        src, dst = kvdgen.random_table(5000, 6000, 6000, seed=3)
        info = pull_and_wait(pair, src, dst)
        assert info["runs"] > 2016
        assert_layers_equal(pair.download_dst(), pair.expected(src, dst))
        # again (slot reuse with an already-grown buffer)
        src2, dst2 = kvdgen.random_table(4000, 6000, 6000, seed=4)
        pre = pair.download_dst()
        pull_and_wait(pair, src2, dst2)
        assert_layers_equal(pair.download_dst(), pair.expected(src2, dst2, pre))
    finally:
        pair.close()


def test_n_zero_completes_without_bytes():
    pair = make_pair(C1, C1, seed=8)
    try:
        info = pull_and_wait(pair, [], [])
        assert info["bytes"] == 0 and info["launches"] == 1
        assert_layers_equal(pair.download_dst(), pair.dst_host)
    finally:
        pair.close()


@pytest.mark.parametrize("src,dst,status", [
    ([0, 64], [1, 2], kvd.ERANGE), ([0, 1], [1, 64], kvd.ERANGE), ([-1], [3], kvd.ERANGE),
    ([0, 1], [3, 3], kvd.EINVAL),
])
def test_errors_change_nothing(src, dst, status):
    pair = make_pair(C1, C1, seed=9)
    try:
        with pytest.raises(kvd.KvdError) as ei:
            pair.peer.pull(next_request_id(), src, dst)
        assert ei.value.status == status
        torch.cuda.synchronize()
        assert_layers_equal(pair.download_dst(), pair.dst_host)
    finally:
        pair.close()


def test_busy_and_unknown_request():
    pair = make_pair(C1, C1, seed=10)
    try:
        rid = next_request_id()
        src, dst = kvdgen.contiguous_table(4)
        pair.peer.pull(rid, src, dst)
        with pytest.raises(kvd.KvdError) as ei:
            pair.peer.pull(rid, src, dst)
        assert ei.value.status == kvd.EBUSY
        pair.peer.wait(rid)
        with pytest.raises(kvd.KvdError) as ei:
            pair.peer.poll(rid)                       # retired after done
        assert ei.value.status == kvd.EINVAL
        pair.peer.pull(rid, src, dst)                 # id may be reused
        pair.peer.wait(rid)
    finally:
        pair.close()


def test_incompatible_caches_rejected():
    a = make_pair(C1, C1, seed=11)
    try:
        other = kvdgen.CacheGeom(2, 2, 64, 8, 64, kvdgen.FP16)      # block_size differs
        from gpu_helpers import cache_for
        c = cache_for(other, 0)
        with pytest.raises(kvd.KvdError) as ei:
            c.open_peer(a.src.export())
        assert ei.value.status == kvd.ELAYOUT
        c.close()
    finally:
        a.close()


def test_many_requests_in_flight_then_poll():
    """Several requests on one stream, polled afterwards in reverse order."""
    g = kvdgen.CacheGeom(2, 2, 64, 16, 256, kvdgen.FP16)
    pair = make_pair(g, g, seed=12)
    try:
        tables = kvdgen.disjoint_fragmented_tables([16, 5, 30, 1, 9, 40], 256, 256, seed=1)
        rids = []
        for s, d in tables:
            rid = next_request_id()
            pair.peer.pull(rid, s, d)
            rids.append(rid)
        for rid in reversed(rids):
            pair.peer.wait(rid)
        exp = pair.dst_host
        for s, d in tables:
            exp = pair.expected(s, d, exp)
        assert_layers_equal(pair.download_dst(), exp)
    finally:
        pair.close()


def test_completion_flag_never_precedes_data():
    """P4: the first time kvd_poll_done returns 1 the host immediately reads
    the destination blocks on ANOTHER stream; they must already hold the
    pulled bytes.  Random n <= 64, C1-like geometry, thousands of pulls."""
    g = kvdgen.CacheGeom(2, 2, 64, 16, 256, kvdgen.FP16)
    pair = make_pair(g, g, seed=13)
    side = torch.cuda.Stream()
    rng = np.random.default_rng(0)
    span = pair.src.span_bytes
    try:
        src_view = [torch.from_numpy(h).view(2, 256, span) for h in pair.src_host]
        for it in range(3000):
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
            for l in range(g.num_layers):
                want = src_view[l][:, torch.from_numpy(s).long()]
                assert torch.equal(got[l], want), f"iteration {it} layer {l}: flag before data"
    finally:
        pair.close()


@pytest.mark.parametrize("single_allocation,devs", [(False, (0, 0)), (True, (0, 0)),
                                                    (False, (0, 1))])
def test_c2_full_size_vs_oracle(single_allocation, devs):
    """C2 at full size (32 layers x 32 heads x 128, 8K tokens = 4 GiB out of
    8 GiB pools) in the launch configuration bench.py times (N = 1 loopback:
    LSU32; N >= 2 over NVLink: the auto TMA ring), compared element by element
    with the CPU oracle: every byte of every layer of the decode cache --
    pulled blocks and untouched ones -- equals the oracle's result on host
    copies of the same inputs (layers split over host threads)."""
    from concurrent.futures import ThreadPoolExecutor
    from gpu_helpers import cache_for
    from oracle import oracle
    if max(devs) >= torch.cuda.device_count():
        pytest.skip("needs two GPUs")
    g = kvdgen.C2
    n = kvdgen.blocks_for(kvdgen.C2_TOKENS, g.block_size)
    src = cache_for(g, devs[0], single_allocation)
    dst = cache_for(g, devs[1], single_allocation)
    for l in range(g.num_layers):
        kvdgen.torch_fill_random_(src.layers[l], 1000 + l)
        kvdgen.torch_fill_random_(dst.layers[l], 2000 + l)
    torch.cuda.synchronize(devs[0])
    torch.cuda.synchronize(devs[1])
    # the oracle's inputs: host copies of exactly what the kernel reads / overwrites
    src_host = [t.cpu().numpy() for t in src.layers]
    pre_host = [t.cpu().numpy() for t in dst.layers]
    peer = dst.open_peer(src.export())
    try:
        s_ids, d_ids = kvdgen.fragmented_table(n, g.num_blocks, g.num_blocks, seed=1)
        rid = next_request_id()
        peer.pull(rid, s_ids, d_ids)
        peer.wait(rid)
        info = peer.info()
        assert info["bytes"] == 4 * 2**30
        assert info["variant"] == (4 if devs[0] != devs[1] else 2)   # the bench's movers
        torch.cuda.synchronize(devs[1])

        def layer(l):
            exp = [pre_host[l]]
            rc = oracle.pull([src_host[l]], g.stride, g.num_blocks, exp, g.stride, g.num_blocks,
                             g.num_kv_heads, g.head_dim, g.block_size, g.elem_bytes, s_ids, d_ids)
            assert rc == oracle.OK
            got = dst.layers[l].cpu().numpy()
            if not np.array_equal(got, exp[0]):
                bad = np.flatnonzero(got != exp[0])
                return f"layer {l}: {bad.size} bytes differ, first at {bad[0]}"
            return None

        with ThreadPoolExecutor(8) as ex:
            errs = [e for e in ex.map(layer, range(g.num_layers)) if e]
        assert not errs, errs[:4]
    finally:
        peer.close()
        dst.close()
        src.close()


def test_c4_shard_full_size_bit_exact():
    """C4 shard (80 layers x 2 heads x 128, bf16, 8K tokens = 640 MiB) fully
    compared with the oracle on host copies."""
    g = kvdgen.C4
    n = kvdgen.blocks_for(kvdgen.C4_TOKENS, g.block_size)
    pair = make_pair(g, g, seed=14)
    try:
        s_ids, d_ids = kvdgen.fragmented_table(n, g.num_blocks, g.num_blocks, seed=4)
        info = pull_and_wait(pair, s_ids, d_ids)
        assert info["bytes"] == 671_088_640
        assert_layers_equal(pair.download_dst(), pair.expected(s_ids, d_ids))
    finally:
        pair.close()


@pytest.mark.gpu2
def test_two_gpus_same_process():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    pair = make_pair(C1.with_blocks(512), C1.with_blocks(512), seed=15, src_dev=0, dst_dev=1)
    try:
        for kind in ("contiguous", "fragmented", "random"):
            src, dst = _tables(kind, 300, 512, 512, seed=3)
            pre = pair.download_dst()
            torch.cuda.set_device(1)
            pull_and_wait(pair, src, dst)
            assert_layers_equal(pair.download_dst(), pair.expected(src, dst, pre))
    finally:
        torch.cuda.set_device(0)
        pair.close()


@pytest.mark.parametrize("kind", ["contiguous", "fragmented", "random"])
def test_push_variant_bit_exact(kind):
    """§8 f2: the push variant (kernel on the prefill side storing into the
    imported decode cache) gives the oracle's result too."""
    pair = make_pair(C1, C1, seed=16)
    try:
        # open the reverse binding: local = prefill cache, imported = decode cache
        rev = pair.src.open_peer(pair.dst.export())
        src, dst = _tables(kind, N_C1, 64, 64, seed=6)
        rid = next_request_id()
        rev.push(rid, src, dst)
        rev.wait(rid)
        assert rev.info()["bytes"] == N_C1 * 2 * 2 * 4096
        assert_layers_equal(pair.download_dst(), pair.expected(src, dst))
        rev.close()
    finally:
        pair.close()


@pytest.mark.gpu2
def test_push_two_gpus():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    g = kvdgen.CacheGeom(4, 8, 128, 16, 300, kvdgen.FP16)
    pair = make_pair(g, g, seed=17, src_dev=0, dst_dev=1)
    try:
        rev = pair.src.open_peer(pair.dst.export())
        src, dst = kvdgen.fragmented_table(200, 300, 300, seed=2)
        rid = next_request_id()
        rev.push(rid, src, dst)
        rev.wait(rid)
        assert_layers_equal(pair.download_dst(), pair.expected(src, dst))
        rev.close()
    finally:
        pair.close()


@pytest.mark.parametrize("threads,stages,ctas", [(32, 2, 1), (96, 4, 0), (256, 2, 5), (64, 8, 3)])
@pytest.mark.parametrize("kind", ["fragmented", "random", "contiguous"])
def test_tma_ring_shapes(threads, stages, ctas, kind):
    """TMA mover: ring depth, pipes per CTA and grid size never change the
    bytes (ragged tiles, more tiles than pipes, fewer tiles than pipes)."""
    g = kvdgen.CacheGeom(3, 4, 64, 16, 128, kvdgen.FP16)
    pair = make_pair(g, g, seed=18)
    try:
        pair.peer.set(kvd.OPT_VARIANT, kvd.VARIANT_TMA).set(kvd.OPT_THREADS, threads)
        pair.peer.set(kvd.OPT_STAGES, stages).set(kvd.OPT_MAX_CTAS, ctas)
        pair.peer.set(kvd.OPT_TILE_BYTES, 3072)
        src, dst = _tables(kind, 77, 128, 128, seed=threads)
        info = pull_and_wait(pair, src, dst)
        assert info["variant"] == kvd.VARIANT_TMA
        assert_layers_equal(pair.download_dst(), pair.expected(src, dst))
    finally:
        pair.close()


def test_tma_rejects_oversized_ring():
    pair = make_pair(C1, C1, seed=19)
    try:
        pair.peer.set(kvd.OPT_VARIANT, kvd.VARIANT_TMA).set(kvd.OPT_THREADS, 256)
        pair.peer.set(kvd.OPT_STAGES, 8).set(kvd.OPT_TILE_BYTES, 8192)   # 8 x 8 x 8 KiB > 225 KiB
        with pytest.raises(kvd.KvdError) as ei:
            pair.peer.pull(next_request_id(), [0], [1])
        assert ei.value.status == kvd.EINVAL
        with pytest.raises(kvd.KvdError) as ei:
            pair.peer.set(kvd.OPT_THREADS, 1024)             # above the 512-thread bound
        assert ei.value.status == kvd.EINVAL
    finally:
        pair.close()


@pytest.mark.gpu2
def test_tma_two_gpus_c4_shard():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    g = kvdgen.C4.with_blocks(600)
    pair = make_pair(g, g, seed=20, src_dev=0, dst_dev=1)
    try:
        pair.peer.set(kvd.OPT_VARIANT, kvd.VARIANT_TMA)
        src, dst = kvdgen.fragmented_table(512, 600, 600, seed=4)
        pull_and_wait(pair, src, dst)
        assert_layers_equal(pair.download_dst(), pair.expected(src, dst))
    finally:
        pair.close()


@pytest.mark.gpu2
@pytest.mark.parametrize("src_dev,dst_dev", [(3, 0), (2, 1), (1, 3)])
def test_any_pair_over_nvswitch(src_dev, dst_dev):
    """NVSwitch is uniform: any prefill GPU -> any decode GPU (SURVEY §8 d,
    C2 "also any i -> j"), auto mover, bit-exact."""
    if max(src_dev, dst_dev) >= torch.cuda.device_count():
        pytest.skip("needs four GPUs")
    g = C1.with_blocks(256)
    pair = make_pair(g, g, seed=40 + src_dev * 4 + dst_dev, src_dev=src_dev, dst_dev=dst_dev)
    try:
        s, d = kvdgen.fragmented_table(120, 256, 256, seed=src_dev * 4 + dst_dev)
        pull_and_wait(pair, s, d)
        assert_layers_equal(pair.download_dst(), pair.expected(s, d))
    finally:
        pair.close()


@pytest.mark.parametrize("variant", [kvd.VARIANT_AUTO, kvd.VARIANT_TMA, kvd.VARIANT_LSU32])
def test_back_to_back_pulls_keep_stream_order(variant):
    """Pulls are launched with programmatic dependent launch; a second pull
    into the SAME destination blocks right behind the first (write after
    write) must still land after it, and a torch kernel zeroing the
    destination before them must land before both."""
    g = C1.with_blocks(512)
    pair = make_pair(g, g, seed=41)
    try:
        pair.peer.set(kvd.OPT_VARIANT, variant)
        rng = np.random.default_rng(3)
        d = rng.choice(512, size=200, replace=False).astype(np.int32)
        s1 = rng.choice(512, size=200, replace=False).astype(np.int32)
        s2 = rng.choice(512, size=200, replace=False).astype(np.int32)
        st = torch.cuda.Stream()
        for _ in range(5):
            with torch.cuda.stream(st):
                for t in pair.dst.layers:
                    t.zero_()
            r1, r2 = next_request_id(), next_request_id()
            pair.peer.pull(r1, s1, d, st)
            pair.peer.pull(r2, s2, d, st)
            pair.peer.wait(r1)
            pair.peer.wait(r2)
            st.synchronize()
            zero = [np.zeros_like(h) for h in pair.dst_host]
            assert_layers_equal(pair.download_dst(), pair.expected(s2, d, zero))
    finally:
        pair.close()


@pytest.mark.parametrize("early", [0, 2, 8])
def test_early_source_reads_keep_destination_order(early):
    """KVD_OPT_EARLY_LOADS: a TMA pull may read its SOURCE before the kernel
    ahead of it on the stream has finished, but every store into the
    destination still follows that kernel: a pull right behind another pull
    into the same blocks (write after write), behind a kernel zeroing the
    destination, lands last -- for every early-read depth."""
    g = kvdgen.CacheGeom(4, 8, 128, 16, 512, kvdgen.FP16)      # 32 KiB spans
    pair = make_pair(g, g, seed=42)
    try:
        pair.peer.set(kvd.OPT_VARIANT, kvd.VARIANT_TMA).set(kvd.OPT_EARLY_LOADS, early)
        rng = np.random.default_rng(4)
        d = rng.choice(512, size=300, replace=False).astype(np.int32)
        st = torch.cuda.Stream()
        for _ in range(5):
            s1 = rng.choice(512, size=300, replace=False).astype(np.int32)
            s2 = rng.choice(512, size=300, replace=False).astype(np.int32)
            with torch.cuda.stream(st):
                for t in pair.dst.layers:
                    t.zero_()
            r1, r2 = next_request_id(), next_request_id()
            pair.peer.pull(r1, s1, d, st)
            pair.peer.pull(r2, s2, d, st)
            pair.peer.wait(r1)
            pair.peer.wait(r2)
            st.synchronize()
            zero = [np.zeros_like(h) for h in pair.dst_host]
            assert_layers_equal(pair.download_dst(), pair.expected(s2, d, zero))
    finally:
        pair.close()


def test_strict_order_chains_pulls():
    """KVD_OPT_EARLY_LOADS = 0 is strict stream order for the source too: a
    pull whose SOURCE is the destination of the pull right before it on the
    same stream (A -> B, then B -> C) reads the bytes the first one wrote."""
    g = kvdgen.CacheGeom(4, 8, 128, 16, 256, kvdgen.FP16)
    ab = make_pair(g, g, seed=43)
    from gpu_helpers import cache_for
    c = cache_for(g, 0)
    try:
        bc = c.open_peer(ab.dst.export())
        for p in (ab.peer, bc):
            p.set(kvd.OPT_VARIANT, kvd.VARIANT_TMA).set(kvd.OPT_EARLY_LOADS, 0)
        s, d = kvdgen.fragmented_table(200, 256, 256, seed=8)
        s2, d2 = kvdgen.fragmented_table(200, 256, 256, seed=9)
        st = torch.cuda.Stream()
        for t in c.layers:
            t.zero_()
        torch.cuda.synchronize()
        r1, r2 = next_request_id(), next_request_id()
        ab.peer.pull(r1, s, d, st)
        bc.pull(r2, d[:150], d2[:150], st)     # reads blocks the first pull writes
        ab.peer.wait(r1)
        bc.wait(r2)
        st.synchronize()
        mid = ab.expected(s, d)
        from oracle import oracle
        want = [np.zeros(c.layer_bytes, np.uint8) for _ in range(g.num_layers)]
        rc = oracle.pull(mid, g.stride, g.num_blocks, want, g.stride, g.num_blocks,
                         g.num_kv_heads, g.head_dim, g.block_size, g.elem_bytes, d[:150], d2[:150])
        assert rc == oracle.OK
        assert_layers_equal([t.cpu().numpy() for t in c.layers], want)
        bc.close()
    finally:
        c.close()
        ab.close()
