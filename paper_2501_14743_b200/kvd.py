"""Thin ctypes binding of the C ABI in include/kvd.h (argument marshalling
only: every step of the pull runs in libkvd.so -- host core + sm_100a
kernels).  Function names are the C names; a negative kvd_status raises
``KvdError`` carrying the status and kvd_last_error().

There is no CPU fallback: if libkvd.so is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes
import os
import threading
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KVD_LIB_PATH") or os.path.join(_HERE, "libkvd.so")   # override: A/B builds

OK, EINVAL, ERANGE, ELAYOUT, EHANDLE, ECUDA, ENOMEM, EBUSY, ESTATE = 0, -1, -2, -3, -4, -5, -6, -7, -8
FP16, BF16, FP8, FP32 = 0, 1, 2, 3
VARIANT_AUTO, VARIANT_LSU, VARIANT_LSU32, VARIANT_CE, VARIANT_TMA = 0, 1, 2, 3, 4
MEM_AUTO, MEM_POSIX_FD, MEM_FABRIC = 0, 1, 8
OPT_MAX_CTAS, OPT_TILE_BYTES, OPT_COALESCE, OPT_VARIANT, OPT_THREADS, OPT_STAGES = 0, 1, 2, 3, 4, 5
OPT_AUDIT, OPT_TIMING, OPT_STREAMS, OPT_EARLY_LOADS, OPT_ENGINE = 6, 7, 8, 9, 10

EXPORTED = (
    "kvd_layout_geometry", "kvd_plan", "kvd_blob_info", "kvd_register_cache",
    "kvd_unregister_cache", "kvd_mem_alloc", "kvd_mem_free", "kvd_export_handle", "kvd_open_peer",
    "kvd_open_peer_heads",
    "kvd_close_peer",
    "kvd_peer_set", "kvd_pull", "kvd_push", "kvd_pull_batch", "kvd_poll_done", "kvd_wait_done",
    "kvd_poll_many",
    "kvd_last_pull_info", "kvd_peer_audit", "kvd_peer_kernel_time", "kvd_peer_device_time",
    "kvd_peer_spans", "kvd_peer_calibrate",
    "kvd_stream_wait",
    "kvd_poll_released",
    "kvd_gather", "kvd_scatter", "kvd_strerror", "kvd_last_error", "kvd_abi_version",
)


class kvd_layout(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_uint32), ("num_kv_heads", ctypes.c_uint32),
                ("head_dim", ctypes.c_uint32), ("block_size", ctypes.c_uint32),
                ("num_blocks", ctypes.c_uint32), ("dtype", ctypes.c_uint32),
                ("stride", ctypes.c_int64 * 5)]


class kvd_geometry(ctypes.Structure):
    _fields_ = [("span_bytes", ctypes.c_uint64), ("block_stride_bytes", ctypes.c_int64),
                ("plane_stride_bytes", ctypes.c_int64), ("layer_bytes", ctypes.c_uint64),
                ("elem_bytes", ctypes.c_uint32), ("kv_adjacent", ctypes.c_uint32)]


class kvd_run(ctypes.Structure):
    _fields_ = [("src_start", ctypes.c_int32), ("dst_start", ctypes.c_int32),
                ("len", ctypes.c_uint32)]


class kvd_pull_info(ctypes.Structure):
    _fields_ = [("request_id", ctypes.c_uint64), ("bytes", ctypes.c_uint64),
                ("blocks", ctypes.c_uint32), ("runs", ctypes.c_uint32),
                ("segments", ctypes.c_uint64), ("tiles", ctypes.c_uint64),
                ("ctas", ctypes.c_uint32), ("threads", ctypes.c_uint32),
                ("variant", ctypes.c_uint32), ("launches", ctypes.c_uint32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class kvd_span(ctypes.Structure):
    _fields_ = [("request_id", ctypes.c_uint64), ("start_ns", ctypes.c_uint64),
                ("wait_ns", ctypes.c_uint64), ("end_ns", ctypes.c_uint64)]


class KvdError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: status {status} ({detail})")
        self.status = status


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

# The ABI version is checked before any other symbol is bound, so a stale
# library fails here with a clear message rather than with AttributeError.
ABI_VERSION = 3     # include/kvd.h KVD_ABI_VERSION this binding was written against
_lib.kvd_abi_version.argtypes = []
_lib.kvd_abi_version.restype = ctypes.c_int
if _lib.kvd_abi_version() != ABI_VERSION:
    raise ImportError(f"{LIB_PATH} has ABI {_lib.kvd_abi_version()}, the binding expects "
                      f"{ABI_VERSION}: rebuild it (__graft_entry__.build())")

_p = ctypes.c_void_p
_u32, _u64, _i32, _i64 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32, ctypes.c_int64
_pi32 = ctypes.POINTER(ctypes.c_int32)

_SIGS = {
    "kvd_layout_geometry": [ctypes.POINTER(kvd_layout), ctypes.POINTER(kvd_geometry)],
    "kvd_plan": [_pi32, _pi32, _u32, _u32, _u32, ctypes.c_int, ctypes.POINTER(kvd_run), _u32,
                 ctypes.POINTER(_u32)],
    "kvd_blob_info": [_p, ctypes.c_size_t, ctypes.POINTER(kvd_layout), ctypes.POINTER(_i32),
                      ctypes.POINTER(_i64), ctypes.POINTER(_u32)],
    "kvd_register_cache": [ctypes.c_int, ctypes.POINTER(kvd_layout), ctypes.POINTER(_p),
                           ctypes.POINTER(_p)],
    "kvd_unregister_cache": [_p],
    "kvd_mem_alloc": [ctypes.c_int, _u64, ctypes.c_int, ctypes.POINTER(_p), ctypes.POINTER(_u64),
                      ctypes.POINTER(ctypes.c_int)],
    "kvd_mem_free": [_p],
    "kvd_export_handle": [_p, _p, ctypes.POINTER(ctypes.c_size_t)],
    "kvd_open_peer": [_p, _p, ctypes.c_size_t, ctypes.POINTER(_p)],
    "kvd_open_peer_heads": [_p, _p, ctypes.c_size_t, _u32, ctypes.POINTER(_p)],
    "kvd_close_peer": [_p],
    "kvd_peer_set": [_p, ctypes.c_int, _i64],
    # hot path: block-id arrays passed as raw addresses (no ctypes pointer objects)
    "kvd_pull": [_p, _u64, _p, _p, _u32, _p],
    "kvd_push": [_p, _u64, _p, _p, _u32, _p],
    "kvd_pull_batch": [_p, _u32, _p, _p, _p, _p, _p],
    "kvd_poll_done": [_p, _u64, ctypes.POINTER(ctypes.c_int)],
    "kvd_wait_done": [_p, _u64, _i64],
    "kvd_poll_many": [_p, _p, _u32, _p, ctypes.POINTER(_u32)],
    "kvd_last_pull_info": [_p, ctypes.POINTER(kvd_pull_info)],
    "kvd_peer_audit": [_p, ctypes.POINTER(_u64)],
    "kvd_poll_released": [_p, _p, _u32, ctypes.POINTER(_u32)],
    "kvd_peer_kernel_time": [_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_u64)],
    "kvd_peer_device_time": [_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_u64)],
    "kvd_peer_spans": [_p, _p, _u32, ctypes.POINTER(_u32)],
    "kvd_peer_calibrate": [_p, _u64, _u32, _u32, _u32, ctypes.POINTER(ctypes.c_double)],
    "kvd_stream_wait": [_p, _p],
    "kvd_gather": [_p, _pi32, _u32, _p, _p],
    "kvd_scatter": [_p, _pi32, _u32, _p, _p],
}
for _name, _args in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = ctypes.c_int
_lib.kvd_strerror.argtypes = [ctypes.c_int]
_lib.kvd_strerror.restype = ctypes.c_char_p
_lib.kvd_last_error.argtypes = []
_lib.kvd_last_error.restype = ctypes.c_char_p


def _check(status: int, where: str) -> int:
    if status < 0:
        raise KvdError(status, where, _lib.kvd_last_error().decode(errors="replace"))
    return status


def _ids(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))


def _ptr_i32(a: np.ndarray):
    return a.ctypes.data_as(_pi32) if a.size else None


def make_layout(num_layers, num_kv_heads, head_dim, block_size, num_blocks, dtype=FP16,
                stride=(0, 0, 0, 0, 0)) -> kvd_layout:
    L = kvd_layout(num_layers, num_kv_heads, head_dim, block_size, num_blocks, dtype)
    for k in range(5):
        L.stride[k] = int(stride[k])
    return L


# ----------------------------------------------------------------------------
# the ABI, one function per C entry point
# ----------------------------------------------------------------------------

def kvd_abi_version() -> int:
    return _lib.kvd_abi_version()


def kvd_strerror(status: int) -> str:
    return _lib.kvd_strerror(status).decode()


def kvd_last_error() -> str:
    return _lib.kvd_last_error().decode(errors="replace")


def kvd_layout_geometry(layout: kvd_layout) -> kvd_geometry:
    g = kvd_geometry()
    _check(_lib.kvd_layout_geometry(ctypes.byref(layout), ctypes.byref(g)), "kvd_layout_geometry")
    return g


def kvd_plan(src_ids, dst_ids, src_num_blocks: int, dst_num_blocks: int,
             coalesce: bool = True) -> np.ndarray:
    """Returns an (m, 3) int64 array of runs (src_start, dst_start, len)."""
    s, d = _ids(src_ids), _ids(dst_ids)
    if s.size != d.size:
        raise ValueError("src_ids and dst_ids differ in length")
    cap = max(1, s.size)
    runs = (kvd_run * cap)()
    m = _u32(0)
    _check(_lib.kvd_plan(_ptr_i32(s), _ptr_i32(d), s.size, src_num_blocks, dst_num_blocks,
                         1 if coalesce else 0, runs, cap, ctypes.byref(m)), "kvd_plan")
    return np.array([(runs[i].src_start, runs[i].dst_start, runs[i].len) for i in range(m.value)],
                    dtype=np.int64).reshape(-1, 3)


def kvd_blob_info(blob: bytes):
    L = kvd_layout()
    dev, pid, na = _i32(0), _i64(0), _u32(0)
    _check(_lib.kvd_blob_info(blob, len(blob), ctypes.byref(L), ctypes.byref(dev),
                              ctypes.byref(pid), ctypes.byref(na)), "kvd_blob_info")
    return L, dev.value, pid.value, na.value


def kvd_register_cache(device: int, layout: kvd_layout, layer_base_dev: Sequence[int]) -> int:
    arr = (_p * len(layer_base_dev))(*[int(b) for b in layer_base_dev])
    h = _p()
    _check(_lib.kvd_register_cache(int(device), ctypes.byref(layout), arr, ctypes.byref(h)),
           "kvd_register_cache")
    return h.value


def kvd_unregister_cache(cache: int) -> None:
    _check(_lib.kvd_unregister_cache(cache), "kvd_unregister_cache")


def kvd_mem_alloc(device: int, nbytes: int, kind: int = MEM_AUTO):
    """§8 f3 groundwork: exportable VMM memory.  Returns (ptr, size, kind)."""
    ptr, size, k = _p(), _u64(0), ctypes.c_int(0)
    _check(_lib.kvd_mem_alloc(int(device), int(nbytes), int(kind), ctypes.byref(ptr),
                              ctypes.byref(size), ctypes.byref(k)), "kvd_mem_alloc")
    return ptr.value, size.value, k.value


def kvd_mem_free(ptr: int) -> None:
    _check(_lib.kvd_mem_free(ptr), "kvd_mem_free")


def kvd_export_handle(cache: int) -> bytes:
    n = ctypes.c_size_t(0)
    st = _lib.kvd_export_handle(cache, None, ctypes.byref(n))
    if st not in (OK, ENOMEM):
        _check(st, "kvd_export_handle")
    buf = ctypes.create_string_buffer(n.value)
    _check(_lib.kvd_export_handle(cache, buf, ctypes.byref(n)), "kvd_export_handle")
    return buf.raw[:n.value]


def kvd_open_peer(local_dst: int, blob: bytes) -> int:
    h = _p()
    _check(_lib.kvd_open_peer(local_dst, blob, len(blob), ctypes.byref(h)), "kvd_open_peer")
    return h.value


def kvd_open_peer_heads(local_dst: int, blob: bytes, head_offset: int) -> int:
    """§8 f4: bind a prefill shard with fewer KV heads to a head slice."""
    h = _p()
    _check(_lib.kvd_open_peer_heads(local_dst, blob, len(blob), head_offset, ctypes.byref(h)),
           "kvd_open_peer_heads")
    return h.value


def kvd_close_peer(peer: int) -> None:
    _check(_lib.kvd_close_peer(peer), "kvd_close_peer")


def kvd_peer_set(peer: int, option: int, value: int) -> None:
    _check(_lib.kvd_peer_set(peer, option, int(value)), "kvd_peer_set")


_from_buffer = ctypes.c_char.from_buffer
_addressof = ctypes.addressof
_I32 = np.dtype(np.int32)


def _addr(a: np.ndarray):
    """Data address of a C-contiguous array (None when empty).  The buffer
    protocol is ~3x cheaper than __array_interface__ per call, which matters
    on the per-request path (C1 latency through Python)."""
    if not a.size:
        return None
    try:
        return _addressof(_from_buffer(a))
    except (TypeError, ValueError):      # read-only buffer
        return a.__array_interface__["data"][0]


def _ids_fast(a) -> np.ndarray:
    if type(a) is np.ndarray and a.dtype is _I32 and a.ndim == 1 and a.flags.c_contiguous:
        return a
    return _ids(a)


def kvd_pull(peer: int, request_id: int, src_ids, dst_ids, stream: Optional[int] = None) -> None:
    """`stream`: a cudaStream_t as int (e.g. torch.cuda.current_stream().cuda_stream)."""
    s, d = _ids_fast(src_ids), _ids_fast(dst_ids)
    if s.size != d.size:
        raise ValueError("src_ids and dst_ids differ in length")
    st = _lib.kvd_pull(peer, request_id, _addr(s), _addr(d), s.size, stream or None)
    if st < 0:
        _check(st, "kvd_pull")


def kvd_push(peer: int, request_id: int, src_ids, dst_ids, stream: Optional[int] = None) -> None:
    """Push variant: local blocks src_ids -> remote blocks dst_ids (launch on the local GPU)."""
    s, d = _ids_fast(src_ids), _ids_fast(dst_ids)
    if s.size != d.size:
        raise ValueError("src_ids and dst_ids differ in length")
    st = _lib.kvd_push(peer, request_id, _addr(s), _addr(d), s.size, stream or None)
    if st < 0:
        _check(st, "kvd_push")


def kvd_pull_batch(peer: int, request_ids, tables, stream: Optional[int] = None) -> None:
    """Batched drain: `tables` is a list of (src_ids, dst_ids), one per request id."""
    ids = np.ascontiguousarray(np.asarray(request_ids, dtype=np.uint64).reshape(-1))
    if ids.size != len(tables):
        raise ValueError("one (src_ids, dst_ids) pair per request id")
    srcs = [_ids(s) for s, _ in tables]
    dsts = [_ids(d) for _, d in tables]
    for s, d in zip(srcs, dsts):
        if s.size != d.size:
            raise ValueError("src_ids and dst_ids differ in length")
    offsets = np.zeros(ids.size + 1, dtype=np.uint32)
    offsets[1:] = np.cumsum([s.size for s in srcs])
    s_all = np.ascontiguousarray(np.concatenate(srcs) if srcs else np.zeros(0, np.int32))
    d_all = np.ascontiguousarray(np.concatenate(dsts) if dsts else np.zeros(0, np.int32))
    st = _lib.kvd_pull_batch(peer, ids.size, _addr(ids), _addr(offsets), _addr(s_all),
                             _addr(d_all), stream or None)
    if st < 0:
        _check(st, "kvd_pull_batch")


_done = ctypes.c_int(0)
_done_ref = ctypes.byref(_done)


def kvd_poll_done(peer: int, request_id: int) -> bool:
    if threading.current_thread() is threading.main_thread():
        st = _lib.kvd_poll_done(peer, request_id, _done_ref)   # reuse one out-cell
        if st < 0:
            _check(st, "kvd_poll_done")
        return bool(_done.value)
    done = ctypes.c_int(0)
    _check(_lib.kvd_poll_done(peer, request_id, ctypes.byref(done)), "kvd_poll_done")
    return bool(done.value)


def kvd_poll_many(peer: int, request_ids) -> list:
    """Retire every completed request among `request_ids`; returns those ids.
    All or nothing: an id not in flight (or listed twice) raises KvdError
    before any request is retired."""
    ids = np.ascontiguousarray(np.asarray(request_ids, dtype=np.uint64).reshape(-1))
    done = np.zeros(max(1, ids.size), dtype=np.uint8)
    n = _u32(0)
    _check(_lib.kvd_poll_many(peer, _addr(ids) if ids.size else None, ids.size, _addr(done),
                              ctypes.byref(n)), "kvd_poll_many")
    return [int(x) for x in ids[done[:ids.size] != 0]]


def kvd_wait_done(peer: int, request_id: int, timeout_us: int = 10_000_000) -> None:
    _check(_lib.kvd_wait_done(peer, request_id, timeout_us), "kvd_wait_done")


def kvd_poll_released(cache: int, cap: int = 4096) -> list:
    """Exporter side of Complete(): request ids whose pulls completed since the last call."""
    buf = np.zeros(max(1, cap), dtype=np.uint64)
    n = _u32(0)
    _check(_lib.kvd_poll_released(cache, _addr(buf), cap, ctypes.byref(n)), "kvd_poll_released")
    return [int(x) for x in buf[:n.value]]


def kvd_peer_audit(peer: int) -> int:
    """Bounds-audit violations counted since KVD_OPT_AUDIT was enabled."""
    v = _u64(0)
    _check(_lib.kvd_peer_audit(peer, ctypes.byref(v)), "kvd_peer_audit")
    return v.value


def kvd_peer_kernel_time(peer: int):
    """(summed kernel-only milliseconds, launches) since the previous call (KVD_OPT_TIMING)."""
    ms, n = ctypes.c_double(0), _u64(0)
    _check(_lib.kvd_peer_kernel_time(peer, ctypes.byref(ms), ctypes.byref(n)),
           "kvd_peer_kernel_time")
    return ms.value, n.value


def kvd_peer_device_time(peer: int):
    """(summed %globaltimer kernel spans in ms, requests) retired since the previous call."""
    ms, n = ctypes.c_double(0), _u64(0)
    _check(_lib.kvd_peer_device_time(peer, ctypes.byref(ms), ctypes.byref(n)),
           "kvd_peer_device_time")
    return ms.value, n.value


def kvd_peer_spans(peer: int, cap: int = 4096) -> list:
    """[(request_id, start_ns, wait_ns, end_ns)] of the timed single pulls
    retired since the previous call (%globaltimer of the decode GPU)."""
    buf = (kvd_span * max(1, cap))()
    n = _u32(0)
    _check(_lib.kvd_peer_spans(peer, ctypes.cast(buf, _p), cap, ctypes.byref(n)), "kvd_peer_spans")
    return [(buf[i].request_id, buf[i].start_ns, buf[i].wait_ns, buf[i].end_ns)
            for i in range(n.value)]


def kvd_peer_calibrate(peer: int, nbytes: int, ctas: int = 0, stages: int = 0,
                       reps: int = 3) -> float:
    """Measured link ceiling: GB/s of discarded bulk reads of `nbytes` of the
    peer's source layers (no stores, no block table), `reps` launches."""
    g = ctypes.c_double(0)
    _check(_lib.kvd_peer_calibrate(peer, int(nbytes), int(ctas), int(stages), int(reps),
                                   ctypes.byref(g)), "kvd_peer_calibrate")
    return g.value


def kvd_stream_wait(peer: int, stream: int) -> None:
    """KVD_OPT_STREAMS >= 2: order `stream` after every transfer issued on the peer."""
    _check(_lib.kvd_stream_wait(peer, stream), "kvd_stream_wait")


def kvd_last_pull_info(peer: int) -> kvd_pull_info:
    info = kvd_pull_info()
    _check(_lib.kvd_last_pull_info(peer, ctypes.byref(info)), "kvd_last_pull_info")
    return info


def kvd_gather(cache: int, ids, staging_dev: int, stream: Optional[int] = None) -> None:
    a = _ids(ids)
    _check(_lib.kvd_gather(cache, _ptr_i32(a), a.size, staging_dev, stream or None), "kvd_gather")


def kvd_scatter(cache: int, ids, staging_dev: int, stream: Optional[int] = None) -> None:
    a = _ids(ids)
    _check(_lib.kvd_scatter(cache, _ptr_i32(a), a.size, staging_dev, stream or None),
           "kvd_scatter")
