"""Pins for the oracle's tensor-centric metadata math (§4.1).

Everything here is checked against something other than the oracle itself:
the values the paper prints for Fig. 5 (tests/golden/fig5_worked_example.txt),
brute-force enumeration of tiny layouts, and closed forms.
"""
import itertools
import os
import random

import numpy as np
import pytest

from oracle import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _fig5():
    shape = stride = elem = None
    offsets, spans, block_spans, coalesce_k = [], None, [], []
    with open(os.path.join(GOLDEN, "fig5_worked_example.txt")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if not line:
                continue
            key, *vals = line.split()
            if key == "shape":
                shape = tuple(int(v) for v in vals)
            elif key == "stride":
                stride = tuple(int(v) for v in vals)
            elif key == "elem_bytes":
                elem = int(vals[0])
            elif key == "offset":
                offsets.append((tuple(int(v) for v in vals[:5]), int(vals[5])))
            elif key == "span":
                spans = int(vals[0])
            elif key == "spans_of_block":
                block_spans.append((int(vals[0]), int(vals[1]), int(vals[2])))
            elif key == "coalesce_k":
                coalesce_k.append(([int(v) for v in vals[0].split(",")],
                                   [int(v) for v in vals[1].split(",")], int(vals[2])))
    return shape, stride, elem, offsets, spans, block_spans, coalesce_k


def test_fig5_offsets_python_and_c():
    shape, stride, elem, offsets, *_ = _fig5()
    assert offsets, "golden file parsed"
    for idx, want in offsets:
        assert oracle.element_offset(stride, idx, elem) == want
        assert oracle.c_element_offset(stride, idx, elem) == want


def test_fig5_default_strides_match_paper():
    # Fig. 5's printed stride vector is the default layout for its shape.
    shape, stride, *_ = _fig5()
    B, KV, L, H, D = shape
    assert oracle.default_strides(B, L, H, D) == stride
    assert oracle.c_default_strides(B, L, H, D) == stride


def test_fig5_span_and_block_spans():
    shape, stride, elem, _, span, block_spans, _ = _fig5()
    assert oracle.span_bytes(shape, stride, elem) == span
    for b, k_off, v_off in block_spans:
        assert oracle.block_to_spans(shape, stride, elem, b) == [(k_off, span), (v_off, span)]
    # two disjoint spaces
    (k0, n0), (k1, n1) = oracle.block_to_spans(shape, stride, elem, 8)
    assert k0 + n0 <= k1 or k1 + n1 <= k0


def test_fig5_coalesce_blocks_0_1():
    shape, stride, elem, _, _, _, coalesce_k = _fig5()
    for src, dst, want in coalesce_k:
        streams = oracle.read_transactions(1, shape, stride, shape, stride, elem, src, dst)
        k_stream = streams[0]
        merged = oracle.coalesce(k_stream)
        assert len(merged) == 1 and merged[0].size == want


def test_span_rule_rejects_non_self_contiguous():
    # (L, H, D) with a gap between heads: the L-stride rule would claim a
    # span the sub-tensor does not fill (reading R4 rejects it).
    shape = (4, 2, 2, 2, 4)
    stride = (64, 256, 16, 8, 1)  # H stride 8 > D=4: gaps
    with pytest.raises(ValueError):
        oracle.span_bytes(shape, stride, 2)


def test_span_rule_largest_stride_excludes_kv():
    # KV stride (40960) is the largest overall; the rule must pick L.
    shape = (10, 2, 16, 2, 128)
    stride = oracle.default_strides(10, 16, 2, 128)
    assert max(stride) == stride[1]
    assert oracle.span_bytes(shape, stride, 2) == 16 * 2 * 128 * 2


def _random_layout(rng):
    B = rng.randint(1, 5)
    L = rng.randint(1, 4)
    H = rng.randint(1, 3)
    D = rng.randint(1, 5)
    sub = L * H * D
    inner_orders = list(itertools.permutations([2, 3, 4]))
    order = rng.choice(inner_orders)       # physical order of L, H, D
    shape = (B, 2, L, H, D)
    stride = [0] * 5
    acc = 1
    for k in reversed(order):              # innermost last
        stride[k] = acc
        acc *= shape[k]
    outer = rng.choice(["kv_outer", "b_outer"])
    pad = rng.randint(0, 2) * sub
    if outer == "kv_outer":
        stride[0] = sub + pad
        stride[1] = B * (sub + pad)
    else:
        stride[1] = sub
        stride[0] = 2 * sub + pad
    return shape, tuple(stride)


def test_offsets_injective_and_partition_bruteforce():
    """distinct indices -> distinct offsets; the (block, kv)
    spans tile exactly the bytes of all elements (brute force)."""
    rng = random.Random(1234)
    for _ in range(200):
        shape, stride = _random_layout(rng)
        elem = rng.choice([1, 2, 4])
        seen = {}
        for idx in itertools.product(*[range(s) for s in shape]):
            off = oracle.element_offset(stride, idx, elem)
            assert oracle.c_element_offset(stride, idx, elem) == off
            assert off not in seen
            seen[off] = idx
        span = oracle.span_bytes(shape, stride, elem)
        covered = set()
        for b in range(shape[0]):
            for off, n in oracle.block_to_spans(shape, stride, elem, b):
                rng_bytes = set(range(off, off + n))
                assert not (covered & rng_bytes)
                covered |= rng_bytes
        elem_bytes = set()
        for off in seen:
            elem_bytes |= set(range(off, off + elem))
        assert covered == elem_bytes
        assert span == shape[2] * shape[3] * shape[4] * elem


def test_layer_nbytes_closed_form():
    B, L, H, D = 10, 16, 2, 128
    stride = oracle.default_strides(B, L, H, D)
    assert oracle.layer_nbytes(stride, B, L, H, D, 2) == 2 * B * 2 * L * H * D
    assert oracle.layer_nbytes((0,) * 5, B, L, H, D, 2) == 2 * B * 2 * L * H * D


def test_block_to_spans_out_of_range():
    shape = (10, 2, 16, 2, 128)
    stride = oracle.default_strides(10, 16, 2, 128)
    with pytest.raises(IndexError):
        oracle.block_to_spans(shape, stride, 2, 10)
