"""CPU-only checks of the C-ABI library (no GPU needed):

* libkvd.so loads and exports every function include/kvd.h declares;
* the host-only entry points (kvd_layout_geometry, kvd_plan, kvd_blob_info)
  agree with the oracle (which shares no code with them) on the paper's
  worked example, on brute-force random tables and on error paths;
* GPU entry points fail with a status (not a crash) when no GPU exists.
"""
import os
import random
import re
import subprocess

import numpy as np
import pytest
import torch

import kvdgen
from oracle import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def kvd():
    from paper_2501_14743_b200 import build
    build.build()
    from paper_2501_14743_b200 import kvd as k
    return k


def _header_functions():
    text = open(os.path.join(ROOT, "include", "kvd.h")).read()
    return sorted(set(re.findall(r"KVD_API\s+[\w\s\*]*?\b(kvd_\w+)\s*\(", text)))


def test_header_declares_boundary_calls():
    names = _header_functions()
    for must in ("kvd_register_cache", "kvd_export_handle", "kvd_open_peer", "kvd_pull",
                 "kvd_poll_done"):
        assert must in names


def test_library_exports_every_declared_symbol(kvd):
    out = subprocess.check_output(["nm", "-D", "--defined-only", kvd.LIB_PATH], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    declared = set(_header_functions())
    assert declared <= exported, declared - exported
    assert exported <= declared, exported - declared       # nothing undeclared leaks
    assert set(kvd.EXPORTED) == declared
    assert kvd.kvd_abi_version() == 3


def test_library_has_no_libcudart_or_torch_dependency(kvd):
    out = subprocess.check_output(["ldd", kvd.LIB_PATH], text=True)
    assert "libtorch" not in out and "libcudart" not in out


def test_sm100a_code_in_library(kvd):
    out = subprocess.check_output(["cuobjdump", "-lelf", kvd.LIB_PATH], text=True)
    assert "sm_100a" in out


# -- geometry vs the oracle --------------------------------------------------

def test_geometry_fig5(kvd):
    # Fig. 5: B=10 L=16 H=2 D=128 bf16, strides (4096, 40960, 256, 128, 1)
    L = kvd.make_layout(1, 2, 128, 16, 10, kvd.BF16, (4096, 40960, 256, 128, 1))
    g = kvd.kvd_layout_geometry(L)
    shape, stride = (10, 2, 16, 2, 128), (4096, 40960, 256, 128, 1)
    assert g.span_bytes == oracle.span_bytes(shape, stride, 2) == 8192
    assert g.block_stride_bytes == oracle.element_offset(stride, (1, 0, 0, 0, 0), 2)
    assert g.plane_stride_bytes == oracle.element_offset(stride, (0, 1, 0, 0, 0), 2)
    assert g.layer_bytes == oracle.layer_nbytes(stride, 10, 16, 2, 128, 2)
    assert g.kv_adjacent == 0
    # all-zero strides select the same layout
    g0 = kvd.kvd_layout_geometry(kvd.make_layout(1, 2, 128, 16, 10, kvd.BF16))
    assert (g0.span_bytes, g0.block_stride_bytes, g0.plane_stride_bytes) == (
        g.span_bytes, g.block_stride_bytes, g.plane_stride_bytes)


def test_geometry_block_major_is_kv_adjacent(kvd):
    sub = 16 * 2 * 128
    g = kvd.kvd_layout_geometry(kvd.make_layout(1, 2, 128, 16, 10, kvd.FP16,
                                                (2 * sub, sub, 256, 128, 1)))
    assert g.kv_adjacent == 1 and g.block_stride_bytes == 2 * g.span_bytes


@pytest.mark.parametrize("stride", [
    (4096, 40960, 256, 64, 1),        # H stride leaves gaps
    (4096, 2048, 256, 128, 1),        # KV planes overlap blocks
    (100, 40960, 256, 128, 1),        # block stride smaller than a block
    (4096, 40960, 256, 128, -1),      # negative stride
])
def test_geometry_rejects_bad_layouts(kvd, stride):
    with pytest.raises(kvd.KvdError) as ei:
        kvd.kvd_layout_geometry(kvd.make_layout(1, 2, 128, 16, 10, kvd.FP16, stride))
    assert ei.value.status == kvd.ELAYOUT


def test_geometry_rejects_unaligned_span(kvd):
    with pytest.raises(kvd.KvdError) as ei:   # 1*1*3 fp16 elements = 6 B span
        kvd.kvd_layout_geometry(kvd.make_layout(1, 1, 3, 1, 4, kvd.FP16))
    assert ei.value.status == kvd.ELAYOUT


def test_geometry_random_layouts_match_oracle(kvd):
    rng = random.Random(3)
    for _ in range(300):
        B, L, H, D = rng.randint(1, 6), rng.randint(1, 4), rng.randint(1, 3), 8 * rng.randint(1, 4)
        sub = L * H * D
        if rng.random() < 0.5:
            stride = (sub, B * sub, H * D, D, 1)
        else:
            stride = (2 * sub + 8 * rng.randint(0, 2), sub, H * D, D, 1)
        g = kvd.kvd_layout_geometry(kvd.make_layout(1, H, D, L, B, kvd.FP16, stride))
        shape = (B, 2, L, H, D)
        assert g.span_bytes == oracle.span_bytes(shape, stride, 2)
        assert g.layer_bytes == oracle.layer_nbytes(stride, B, L, H, D, 2)
        assert oracle.block_to_spans(shape, stride, 2, B - 1) == [
            ((B - 1) * g.block_stride_bytes, g.span_bytes),
            ((B - 1) * g.block_stride_bytes + g.plane_stride_bytes, g.span_bytes)]


# -- plan (validate + coalesce) vs the oracle's byte-space coalescing --------

def _segments_from_runs(runs, span, plane, layers=1):
    """Expand block runs into byte segments of the default layout (test-side)."""
    out = []
    for layer in range(layers):
        for kv in range(2):
            for s, d, n in runs:
                out.append((layer, kv, kv * plane + int(s) * span, kv * plane + int(d) * span,
                            int(n) * span))
    return out


def test_plan_matches_oracle_coalesce_random(kvd):
    rng = random.Random(11)
    nb = 40
    shape, stride = (nb, 2, 4, 2, 16), oracle.default_strides(nb, 4, 2, 16)
    span = 4 * 2 * 16 * 2
    for _ in range(1000):
        n = rng.randint(0, 30)
        if rng.random() < 0.5:
            src, dst = rng.sample(range(nb), n), rng.sample(range(nb), n)
        else:
            s0, d0 = rng.randint(0, nb - n), rng.randint(0, nb - n)
            src, dst = list(range(s0, s0 + n)), list(range(d0, d0 + n))
            for _k in range(rng.randint(0, 3)):
                if n > 1:
                    i = rng.randrange(n - 1)
                    dst[i], dst[i + 1] = dst[i + 1], dst[i]
        runs = kvd.kvd_plan(src, dst, nb, nb, coalesce=True)
        ours = sorted(_segments_from_runs(runs, span, nb * span))
        ref = []
        for stream in oracle.read_transactions(1, shape, stride, shape, stride, 2, src, dst):
            ref += [(r.layer, r.kv, r.remote, r.local, r.size) for r in oracle.coalesce(stream)]
        assert ours == sorted(ref)
        # coalesce off: one run per block
        assert len(kvd.kvd_plan(src, dst, nb, nb, coalesce=False)) == n


def test_plan_fig_queue_and_fig5(kvd):
    assert kvd.kvd_plan([0, 1], [5, 6], 12, 12).tolist() == [[0, 5, 2]]
    assert kvd.kvd_plan([0, 1], [5, 9], 12, 12).tolist() == [[0, 5, 1], [1, 9, 1]]
    assert kvd.kvd_plan([0, 1], [0, 1], 10, 10).tolist() == [[0, 0, 2]]


@pytest.mark.parametrize("src,dst,status", [
    ([0, 10], [1, 2], -2), ([0, 1], [1, 10], -2), ([-1], [0], -2), ([0], [-5], -2),
    ([0, 1], [3, 3], -1),
])
def test_plan_errors_match_oracle(kvd, src, dst, status):
    with pytest.raises(kvd.KvdError) as ei:
        kvd.kvd_plan(src, dst, 10, 10)
    assert ei.value.status == status
    # the oracle takes the same decision
    g = kvdgen.CacheGeom(1, 1, 8, 1, 10, kvdgen.FP16)
    layer = np.zeros(oracle.layer_nbytes((0,) * 5, 10, 1, 1, 8, 2), np.uint8)
    rc = oracle.pull([layer], (0,) * 5, 10, [layer.copy()], (0,) * 5, 10, 1, 8, 1, 2,
                     np.array(src, np.int32), np.array(dst, np.int32))
    assert rc == status


def test_plan_duplicate_source_allowed(kvd):
    assert kvd.kvd_plan([3, 3], [0, 1], 10, 10).tolist() == [[3, 0, 1], [3, 1, 1]]


def test_plan_large_fragmented_c2(kvd):
    src, dst = kvdgen.fragmented_table(512, 1024, 1024, seed=1)
    runs = kvd.kvd_plan(src, dst, 1024, 1024)
    assert runs[:, 2].sum() == 512
    brk = sum(1 for i in range(511) if not (src[i + 1] == src[i] + 1 and dst[i + 1] == dst[i] + 1))
    assert len(runs) == brk + 1


# -- blob codec and no-GPU behaviour ------------------------------------------

@pytest.mark.parametrize("blob", [b"", b"KVDB", b"\x00" * 64, b"KVDB" + b"\x01" * 300])
def test_blob_info_rejects_malformed(kvd, blob):
    with pytest.raises(kvd.KvdError) as ei:
        kvd.kvd_blob_info(blob)
    assert ei.value.status == kvd.EHANDLE


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU path")
def test_register_without_gpu_fails_cleanly(kvd):
    L = kvd.make_layout(2, 2, 64, 16, 64)
    with pytest.raises(kvd.KvdError) as ei:
        kvd.kvd_register_cache(0, L, [1 << 20, 1 << 21])
    assert ei.value.status in (kvd.ECUDA, kvd.EINVAL)
    # layout errors are reported before any CUDA call
    with pytest.raises(kvd.KvdError) as ei:
        kvd.kvd_register_cache(0, kvd.make_layout(2, 2, 64, 16, 0), [1 << 20, 1 << 21])
    assert ei.value.status == kvd.ELAYOUT


def test_argument_errors_before_any_cuda_call(kvd):
    """Entry points reject null / out-of-range arguments with the documented
    status on a machine without a GPU too."""
    import ctypes
    lib = kvd._lib
    assert lib.kvd_mem_free(None) == kvd.EINVAL
    p = ctypes.c_void_p()
    assert lib.kvd_mem_alloc(0, 1 << 20, 5, ctypes.byref(p), None, None) == kvd.EINVAL   # bad kind
    assert lib.kvd_mem_alloc(0, 0, 0, ctypes.byref(p), None, None) == kvd.EINVAL         # zero bytes
    assert lib.kvd_mem_alloc(0, 1 << 20, 0, None, None, None) == kvd.EINVAL              # null out
    assert lib.kvd_stream_wait(None, None) == kvd.EINVAL
    nd = ctypes.c_uint32()
    assert lib.kvd_poll_many(None, None, 0, None, ctypes.byref(nd)) == kvd.EINVAL
    ms, n = ctypes.c_double(), ctypes.c_uint64()
    assert lib.kvd_peer_device_time(None, ctypes.byref(ms), ctypes.byref(n)) == kvd.EINVAL
    assert lib.kvd_peer_kernel_time(None, ctypes.byref(ms), ctypes.byref(n)) == kvd.EINVAL
    assert lib.kvd_close_peer(None) == kvd.EINVAL
    assert lib.kvd_unregister_cache(None) == kvd.EINVAL
    assert lib.kvd_peer_set(None, kvd.OPT_STREAMS, 2) == kvd.EINVAL
    assert "invalid argument" in kvd.kvd_strerror(kvd.EINVAL)
