"""oracle/oracle.py -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Plain CPU oracle for KVDirect's pull path (arXiv 2501.14743).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  It shares no code with
``paper_2501_14743_b200/`` (the CUDA path) and imports nothing from it.

Contents, each following a passage of PAPER.md (cited as P:Lnnn):

* ``element_offset``      -- the tensor-centric address rule.
* ``default_strides``     -- Fig. 5's stride pattern (K block tensors first,
                             then V).
* ``span_bytes``          -- the contiguous-span rule, with the
                             self-contiguity reading R4 of DESIGN.md.
* ``block_to_spans``      -- "the two tensors in block 8 are stored as two
                             disjoint 8192 B memory spaces".
* ``read_transactions``   -- one Read(remote span -> local span) per block
                             and K/V tensor, in block-table order, P:L306,
                             P:L373.
* ``coalesce``            -- "A group of transactions can be merged only
                             when the results of both remote and local
                             locations are contiguous".
* ``pull``                -- the copy itself: a ctypes call into
                             ``kvd_oracle.c`` (an element-by-element loop).

Pinning (tests/test_oracle_*.py): Fig. 5 worked example values, fig:queue
merge example, brute-force enumeration on tiny layouts, two loop orders,
and NumPy fancy indexing as the library special case.  Nothing here is
"parity unpinned".
"""

from __future__ import annotations

import ctypes
import functools
import itertools
import os
import subprocess
from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kvd_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, EINVAL, ERANGE = 0, -1, -2

# Dims order of Fig. 5: cache[B][KV][L][H][D].
DIMS = ("B", "KV", "L", "H", "D")


# --------------------------------------------------------------------------
# build / load the C oracle
# --------------------------------------------------------------------------

def build(force: bool = False) -> str:
    """Compile kvd_oracle.c into liboracle.so with plain gcc -O2."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        p_i64 = ctypes.POINTER(ctypes.c_int64)
        p_i32 = ctypes.POINTER(ctypes.c_int32)
        p_ptr = ctypes.POINTER(ctypes.c_void_p)
        for name in ("oracle_pull_blockwise", "oracle_pull_tokenwise"):
            fn = getattr(lib, name)
            fn.restype = ctypes.c_int
            fn.argtypes = [p_ptr, p_i64, ctypes.c_uint32, p_ptr, p_i64, ctypes.c_uint32,
                           ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                           ctypes.c_uint32, p_i32, p_i32, ctypes.c_uint32]
        lib.oracle_pull_heads.restype = ctypes.c_int
        lib.oracle_pull_heads.argtypes = [p_ptr, p_i64, ctypes.c_uint32, ctypes.c_uint32,
                                          p_ptr, p_i64, ctypes.c_uint32, ctypes.c_uint32,
                                          ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                          ctypes.c_uint32, ctypes.c_uint32, p_i32, p_i32,
                                          ctypes.c_uint32]
        lib.oracle_element_offset.restype = ctypes.c_int64
        lib.oracle_element_offset.argtypes = [p_i64, p_i64, ctypes.c_uint32]
        lib.oracle_default_strides.restype = None
        lib.oracle_default_strides.argtypes = [ctypes.c_uint32] * 4 + [p_i64]
        lib.oracle_layer_element_offset.restype = ctypes.c_int64
        lib.oracle_layer_element_offset.argtypes = (
            [p_i64] + [ctypes.c_uint32] * 5 + [ctypes.c_int64] * 5)
        _lib = lib
    return _lib


def _i64(vals):
    arr = (ctypes.c_int64 * len(vals))(*[int(v) for v in vals])
    return arr


# --------------------------------------------------------------------------
# tensor-centric metadata, pure Python
# --------------------------------------------------------------------------

def default_strides(num_blocks: int, block_size: int, num_heads: int, head_dim: int):
    """Fig. 5's layout: the K sub-tensors (L, H, D) of all
    blocks are contiguous, then the V sub-tensors, so
    stride = (L*H*D, B*L*H*D, H*D, D, 1) in Dims order (B, KV, L, H, D)."""
    sub = block_size * num_heads * head_dim
    return (sub, num_blocks * sub, num_heads * head_dim, head_dim, 1)


def element_offset(stride: Sequence[int], index: Sequence[int], elem_bytes: int) -> int:
    """byte offset = (index . stride) * element size."""
    assert len(stride) == len(index)
    return sum(int(i) * int(s) for i, s in zip(index, stride)) * int(elem_bytes)


def span_bytes(shape: Sequence[int], stride: Sequence[int], elem_bytes: int) -> int:
    return _span_bytes(tuple(int(s) for s in shape), tuple(int(s) for s in stride),
                       int(elem_bytes))


@functools.lru_cache(maxsize=4096)
def _span_bytes(shape: Tuple[int, ...], stride: Tuple[int, ...], elem_bytes: int) -> int:
    """"We find the dimension with the largest stride, L, and then
    multiply its shape with the stride" -- taken among the per-block
    dimensions L, H, D (reading R4: the KV stride is larger but is not part
    of a block's sub-tensor).  The sub-tensor must be self-contiguous (its
    element offsets are exactly 0 .. L*H*D-1), otherwise the layout is
    rejected (reading R4); checked here by enumerating every element."""
    inner = [2, 3, 4]  # L, H, D
    # ties in stride occur only next to an extent-1 dimension; the dimension
    # that spans the sub-tensor is then the one with the larger shape (R4)
    d_star = max(inner, key=lambda k: (stride[k], shape[k]))
    span = int(shape[d_star]) * int(stride[d_star]) * int(elem_bytes)
    offs = sorted(
        element_offset([stride[k] for k in inner], idx, 1)
        for idx in itertools.product(*[range(shape[k]) for k in inner]))
    count = int(shape[2]) * int(shape[3]) * int(shape[4])
    if offs != list(range(count)) or span != count * elem_bytes:
        raise ValueError("(L, H, D) sub-tensor is not self-contiguous")
    return span


def block_to_spans(shape, stride, elem_bytes: int, block: int) -> List[Tuple[int, int]]:
    """block b's K and V tensors start at cache[b][kv][0][0][0]
    and each covers span_bytes; returns [(offset, length)] for kv = 0, 1."""
    if not 0 <= block < shape[0]:
        raise IndexError("block id out of range")
    span = span_bytes(shape, stride, elem_bytes)
    return [(element_offset(stride, (block, kv, 0, 0, 0), elem_bytes), span)
            for kv in range(shape[1])]


@dataclass(frozen=True)
class Read:
    """A Read transaction (fig:queue) for one (layer, K/V tensor)."""
    layer: int
    kv: int
    remote: int   # byte offset in the remote (prefill) layer tensor
    local: int    # byte offset in the local (decode) layer tensor
    size: int


def read_transactions(num_layers, src_shape, src_stride, dst_shape, dst_stride,
                      elem_bytes, src_ids, dst_ids) -> List[List[Read]]:
    """Translate Transfer(remote block, local block) calls into byte
    Reads, one per block and K/V tensor, grouped per (layer, kv) stream in
    block-table order (reading R10: coalescing works within a stream)."""
    streams = []
    for layer in range(num_layers):
        for kv in range(2):
            stream = []
            for s, d in zip(src_ids, dst_ids):
                r_off, r_len = block_to_spans(src_shape, src_stride, elem_bytes, s)[kv]
                l_off, l_len = block_to_spans(dst_shape, dst_stride, elem_bytes, d)[kv]
                assert r_len == l_len
                stream.append(Read(layer, kv, r_off, l_off, r_len))
            streams.append(stream)
    return streams


def coalesce(stream: Sequence[Read]) -> List[Read]:
    """pop the Reads in order; merge a Read into the previous one
    only when BOTH its remote and its local location continue the previous
    one's ("both remote and local locations are contiguous")."""
    out: List[Read] = []
    for r in stream:
        if out:
            p = out[-1]
            if (p.layer == r.layer and p.kv == r.kv and p.remote + p.size == r.remote
                    and p.local + p.size == r.local):
                out[-1] = Read(p.layer, p.kv, p.remote, p.local, p.size + r.size)
                continue
        out.append(r)
    return out


# --------------------------------------------------------------------------
# the copy (C element loop)
# --------------------------------------------------------------------------

def _ptrs(arrays):
    return (ctypes.c_void_p * len(arrays))(*[a.ctypes.data for a in arrays])


def pull(src_layers: Sequence[np.ndarray], src_stride, src_num_blocks: int,
         dst_layers: Sequence[np.ndarray], dst_stride, dst_num_blocks: int,
         num_heads: int, head_dim: int, block_size: int, elem_bytes: int,
         src_ids, dst_ids, order: str = "block") -> int:
    """Run the C oracle in place on host byte buffers (one per layer).

    ``src_stride``/``dst_stride`` are element strides in Dims order
    (B, KV, L, H, D); all zeros selects Fig. 5's default layout.
    Returns OK / EINVAL / ERANGE; on error nothing is written."""
    lib = _load()
    assert len(src_layers) == len(dst_layers)
    for a in list(src_layers) + list(dst_layers):
        assert a.flags["C_CONTIGUOUS"]
    src_ids = np.ascontiguousarray(src_ids, dtype=np.int32)
    dst_ids = np.ascontiguousarray(dst_ids, dtype=np.int32)
    assert src_ids.shape == dst_ids.shape
    fn = lib.oracle_pull_blockwise if order == "block" else lib.oracle_pull_tokenwise
    p_i32 = ctypes.POINTER(ctypes.c_int32)
    return fn(_ptrs(src_layers), _i64(src_stride), src_num_blocks,
              _ptrs(dst_layers), _i64(dst_stride), dst_num_blocks,
              len(src_layers), num_heads, head_dim, block_size, elem_bytes,
              src_ids.ctypes.data_as(p_i32), dst_ids.ctypes.data_as(p_i32),
              int(src_ids.shape[0]))


def pull_heads(src_layers, src_stride, src_num_blocks: int, src_heads: int,
               dst_layers, dst_stride, dst_num_blocks: int, dst_heads: int, head_offset: int,
               head_dim: int, block_size: int, elem_bytes: int, src_ids, dst_ids) -> int:
    """§8 f4 TP-resharding pull: source heads land at destination heads
    [head_offset, head_offset + src_heads) (kvd_oracle.c: oracle_pull_heads)."""
    lib = _load()
    src_ids = np.ascontiguousarray(src_ids, dtype=np.int32)
    dst_ids = np.ascontiguousarray(dst_ids, dtype=np.int32)
    p_i32 = ctypes.POINTER(ctypes.c_int32)
    return lib.oracle_pull_heads(
        _ptrs(src_layers), _i64(src_stride), src_num_blocks, src_heads,
        _ptrs(dst_layers), _i64(dst_stride), dst_num_blocks, dst_heads, head_offset,
        len(src_layers), head_dim, block_size, elem_bytes,
        src_ids.ctypes.data_as(p_i32), dst_ids.ctypes.data_as(p_i32), int(src_ids.shape[0]))


def c_element_offset(stride, index, elem_bytes: int) -> int:
    return _load().oracle_element_offset(_i64(stride), _i64(index), elem_bytes)


def c_default_strides(num_blocks, block_size, num_heads, head_dim):
    out = (ctypes.c_int64 * 5)()
    _load().oracle_default_strides(num_blocks, block_size, num_heads, head_dim, out)
    return tuple(out)


def c_layer_element_offset(stride, num_blocks, block_size, num_heads, head_dim,
                           elem_bytes, b, kv, t, h, d) -> int:
    return _load().oracle_layer_element_offset(
        _i64(stride), num_blocks, block_size, num_heads, head_dim, elem_bytes,
        b, kv, t, h, d)


def layer_nbytes(stride, num_blocks, block_size, num_heads, head_dim, elem_bytes) -> int:
    """Bytes one layer tensor occupies: one past its largest element offset."""
    last = c_layer_element_offset(stride, num_blocks, block_size, num_heads, head_dim,
                                  elem_bytes, num_blocks - 1, 1, block_size - 1,
                                  num_heads - 1, head_dim - 1)
    return max(last, 0) + elem_bytes
