"""Pins for the oracle's copy (SURVEY.md §8 row c, P3/P5/P6).

* library special case: NumPy fancy indexing T[:, dst] = S[:, src] on the
  (KV, B, L, H, D) physical layout of Fig. 5, and on a (B, KV, L, H, D)
  layout through a transposed view;
* the two loop orders (block-ordered, token brute force) agree byte for byte;
* invariants I1 (every token's K/V identical), I2 (untouched destination
  blocks unchanged), I3 (source unchanged), I6 (idempotent), I7 (n = 0);
* error paths leave the destination byte-identical;
* random 16-bit words (NaN payloads, -0, subnormals, Inf) survive.
"""
import numpy as np
import pytest

import kvdgen
from oracle import oracle


def _alloc(geom: kvdgen.CacheGeom, seed: int, side: int):
    stride = geom.stride if any(geom.stride) else oracle.default_strides(
        geom.num_blocks, geom.block_size, geom.num_kv_heads, geom.head_dim)
    nbytes = oracle.layer_nbytes(stride, geom.num_blocks, geom.block_size,
                                 geom.num_kv_heads, geom.head_dim, geom.elem_bytes)
    return [kvdgen.random_bytes(nbytes, seed * 1000 + side * 100 + l)
            for l in range(geom.num_layers)]


def _run(sg, dg, src_layers, dst_layers, src_ids, dst_ids, order="block"):
    return oracle.pull(src_layers, sg.stride, sg.num_blocks, dst_layers, dg.stride,
                       dg.num_blocks, sg.num_kv_heads, sg.head_dim, sg.block_size,
                       sg.elem_bytes, src_ids, dst_ids, order=order)


GEOMS = [
    kvdgen.C1,
    kvdgen.CacheGeom(3, 1, 8, 4, 9, kvdgen.FP16),
    kvdgen.CacheGeom(2, 3, 4, 2, 7, kvdgen.FP8),
    kvdgen.CacheGeom(1, 2, 16, 8, 5, kvdgen.FP32),
]


@pytest.mark.parametrize("geom", GEOMS)
def test_numpy_fancy_indexing_default_layout(geom):
    dgeom = geom.with_blocks(geom.num_blocks + 3)
    src = _alloc(geom, 1, 0)
    dst = _alloc(dgeom, 1, 1)
    before = [d.copy() for d in dst]
    src_ids, dst_ids = kvdgen.random_table(min(geom.num_blocks, 6), geom.num_blocks,
                                           dgeom.num_blocks, seed=3)
    assert _run(geom, dgeom, src, dst, src_ids, dst_ids) == oracle.OK
    e = geom.elem_bytes
    for l in range(geom.num_layers):
        shp = (2, geom.num_blocks, geom.block_size, geom.num_kv_heads, geom.head_dim * e)
        dshp = (2, dgeom.num_blocks) + shp[2:]
        S = src[l].reshape(shp)
        T = before[l].reshape(dshp).copy()
        T[:, dst_ids] = S[:, src_ids]
        assert np.array_equal(T.reshape(-1), dst[l])


def test_numpy_fancy_indexing_block_major_layout():
    """(B, KV, L, H, D) physical order (K and V of a block adjacent)."""
    B, L, H, D, e = 6, 4, 2, 8, 2
    sub = L * H * D
    stride = (2 * sub, sub, H * D, D, 1)
    g = kvdgen.CacheGeom(2, H, D, L, B, kvdgen.BF16, stride)
    src = _alloc(g, 5, 0)
    dst = _alloc(g, 5, 1)
    before = [d.copy() for d in dst]
    src_ids = np.array([4, 0, 5], np.int32)
    dst_ids = np.array([1, 2, 3], np.int32)
    assert _run(g, g, src, dst, src_ids, dst_ids) == oracle.OK
    for l in range(2):
        S = src[l].reshape(B, 2, L, H, D * e)
        T = before[l].reshape(B, 2, L, H, D * e).copy()
        T[dst_ids] = S[src_ids]
        assert np.array_equal(T.reshape(-1), dst[l])


def test_mixed_layouts_src_kv_outer_dst_block_major():
    """The paper allows "a different order of these five dimensions"
    (P:L300); the copy is defined element-wise, so mixed layouts work."""
    B, L, H, D, e = 5, 2, 2, 4, 2
    sub = L * H * D
    sg = kvdgen.CacheGeom(1, H, D, L, B, kvdgen.FP16)
    dg = kvdgen.CacheGeom(1, H, D, L, B, kvdgen.FP16, (2 * sub, sub, H * D, D, 1))
    src = _alloc(sg, 9, 0)
    dst = _alloc(dg, 9, 1)
    before = dst[0].copy()
    src_ids = np.array([0, 3], np.int32)
    dst_ids = np.array([4, 1], np.int32)
    assert _run(sg, dg, src, dst, src_ids, dst_ids) == oracle.OK
    S = src[0].reshape(2, B, L, H, D * e)
    T = before.reshape(B, 2, L, H, D * e).copy()
    T[dst_ids] = np.swapaxes(S[:, src_ids], 0, 1)
    assert np.array_equal(T.reshape(-1), dst[0])


@pytest.mark.parametrize("geom", GEOMS)
def test_block_order_equals_token_order(geom):
    src = _alloc(geom, 2, 0)
    d1 = _alloc(geom, 2, 1)
    d2 = [d.copy() for d in d1]
    n = min(geom.num_blocks, 5)
    src_ids, dst_ids = kvdgen.random_table(n, geom.num_blocks, geom.num_blocks, seed=11)
    assert _run(geom, geom, src, d1, src_ids, dst_ids, "block") == oracle.OK
    assert _run(geom, geom, src, d2, src_ids, dst_ids, "token") == oracle.OK
    for a, b in zip(d1, d2):
        assert np.array_equal(a, b)


def test_invariants_c1():
    """I1, I2, I3, I6 on the C1 configuration (256-token request)."""
    g = kvdgen.C1
    n = kvdgen.blocks_for(kvdgen.C1_TOKENS, g.block_size)
    src = _alloc(g, 3, 0)
    src_copy = [s.copy() for s in src]
    dst = _alloc(g, 3, 1)
    before = [d.copy() for d in dst]
    src_ids, dst_ids = kvdgen.fragmented_table(n, g.num_blocks, g.num_blocks, seed=0)
    assert _run(g, g, src, dst, src_ids, dst_ids) == oracle.OK
    e, L, H, D = g.elem_bytes, g.block_size, g.num_kv_heads, g.head_dim
    for l in range(g.num_layers):
        S = src[l].reshape(2, g.num_blocks, L, H, D * e)
        T = dst[l].reshape(2, g.num_blocks, L, H, D * e)
        T0 = before[l].reshape(2, g.num_blocks, L, H, D * e)
        # I1: token q of the prompt lives at (src_ids[q // L], q % L) on the
        # prefill side and at (dst_ids[q // L], q % L) on the decode side.
        for q in range(kvdgen.C1_TOKENS):
            for kv in range(2):
                for h in range(H):
                    assert np.array_equal(T[kv, dst_ids[q // L], q % L, h],
                                          S[kv, src_ids[q // L], q % L, h])
        # I2: blocks not in dst_ids unchanged
        untouched = sorted(set(range(g.num_blocks)) - set(dst_ids.tolist()))
        assert np.array_equal(T[:, untouched], T0[:, untouched])
        # I3: source unchanged
        assert np.array_equal(src[l], src_copy[l])
    # I6: pulling again changes nothing
    snap = [d.copy() for d in dst]
    assert _run(g, g, src, dst, src_ids, dst_ids) == oracle.OK
    for a, b in zip(snap, dst):
        assert np.array_equal(a, b)


def test_n_zero_changes_nothing():
    g = kvdgen.C1
    src = _alloc(g, 4, 0)
    dst = _alloc(g, 4, 1)
    before = [d.copy() for d in dst]
    empty = np.zeros(0, np.int32)
    assert _run(g, g, src, dst, empty, empty) == oracle.OK
    for a, b in zip(before, dst):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("src_ids,dst_ids,rc", [
    ([0, 64], [1, 2], oracle.ERANGE),
    ([0, 1], [1, 64], oracle.ERANGE),
    ([-1, 1], [1, 2], oracle.ERANGE),
    ([0, 1], [3, 3], oracle.EINVAL),
    ([5, 5], [3, 4], oracle.OK),           # duplicate source is allowed (R9)
])
def test_error_paths_leave_destination_untouched(src_ids, dst_ids, rc):
    g = kvdgen.C1
    src = _alloc(g, 6, 0)
    dst = _alloc(g, 6, 1)
    before = [d.copy() for d in dst]
    got = _run(g, g, src, dst, np.array(src_ids, np.int32), np.array(dst_ids, np.int32))
    assert got == rc
    if rc != oracle.OK:
        for a, b in zip(before, dst):
            assert np.array_equal(a, b)


def test_special_float_words_survive():
    """P5: every fp16/bf16 NaN payload, +-Inf, -0 and subnormal is copied
    bit for bit (a float-typed copy would canonicalise NaNs)."""
    g = kvdgen.CacheGeom(1, 1, 256, 16, 8, kvdgen.FP16)
    words = np.arange(65536, dtype=np.uint16)            # all 16-bit patterns
    layer = np.zeros(oracle.layer_nbytes((0,) * 5, 8, 16, 1, 256, 2), np.uint8)
    assert layer.size == 2 * words.size
    layer.view(np.uint16)[:] = words
    dst = [np.zeros_like(layer)]
    ids = np.arange(8, dtype=np.int32)
    assert _run(g, g, [layer], dst, ids, ids[::-1].copy()) == oracle.OK
    S = layer.view(np.uint16).reshape(2, 8, -1)
    T = dst[0].view(np.uint16).reshape(2, 8, -1)
    assert np.array_equal(T[:, ::-1], S)
    assert np.array_equal(np.sort(T.reshape(-1)), words)
