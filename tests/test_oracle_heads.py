"""Pins for the oracle's TP-resharding pull (§8 f4).

* NumPy fancy indexing with a head slice T[:, dst, :, off:off+Hs] = S[:, src]
  (library special case) on the default layout;
* composition: pulling prefill TP=8 shards 2j and 2j+1 into decode TP=4 shard
  j reproduces, byte for byte, a plain pull from an unsharded (TP=4 shaped)
  source whose heads are the two shards' heads side by side;
* src_heads == dst_heads, offset 0 reduces to the plain pull;
* out-of-range head placement and block ids are rejected, nothing written.
"""
import numpy as np
import pytest

import kvdgen
from oracle import oracle

L, D, E = 16, 8, 2


def _layers(nl, nb, heads, seed):
    nbytes = oracle.layer_nbytes((0,) * 5, nb, L, heads, D, E)
    return [kvdgen.random_bytes(nbytes, seed + l) for l in range(nl)]


@pytest.mark.parametrize("hs,hd,off", [(1, 2, 0), (1, 2, 1), (2, 8, 4), (3, 3, 0)])
def test_head_slice_numpy(hs, hd, off):
    nl, nb = 2, 12
    src = _layers(nl, nb, hs, 1)
    dst = _layers(nl, nb, hd, 50)
    before = [d.copy() for d in dst]
    s_ids, d_ids = kvdgen.random_table(7, nb, nb, seed=4)
    rc = oracle.pull_heads(src, (0,) * 5, nb, hs, dst, (0,) * 5, nb, hd, off, D, L, E,
                           s_ids, d_ids)
    assert rc == oracle.OK
    for l in range(nl):
        S = src[l].reshape(2, nb, L, hs, D * E)
        T = before[l].reshape(2, nb, L, hd, D * E).copy()
        T[:, d_ids, :, off:off + hs] = S[:, s_ids]
        assert np.array_equal(T.reshape(-1), dst[l])


def test_tp8_to_tp4_composition():
    nl, nb, hs = 2, 10, 1
    shard0 = _layers(nl, nb, hs, 100)
    shard1 = _layers(nl, nb, hs, 200)
    s_ids, d_ids = kvdgen.random_table(6, nb, nb, seed=9)
    dst = _layers(nl, nb, 2 * hs, 300)
    ref = [d.copy() for d in dst]
    assert oracle.pull_heads(shard0, (0,) * 5, nb, hs, dst, (0,) * 5, nb, 2 * hs, 0, D, L, E,
                             s_ids, d_ids) == oracle.OK
    assert oracle.pull_heads(shard1, (0,) * 5, nb, hs, dst, (0,) * 5, nb, 2 * hs, hs, D, L, E,
                             s_ids, d_ids) == oracle.OK
    # the unsharded source: heads of shard 0 then shard 1, per token
    merged = []
    for l in range(nl):
        a = shard0[l].reshape(2, nb, L, hs, D * E)
        b = shard1[l].reshape(2, nb, L, hs, D * E)
        merged.append(np.ascontiguousarray(np.concatenate([a, b], axis=3)).reshape(-1))
    assert oracle.pull(merged, (0,) * 5, nb, ref, (0,) * 5, nb, 2 * hs, D, L, E,
                       s_ids, d_ids) == oracle.OK
    for a, b in zip(dst, ref):
        assert np.array_equal(a, b)


def test_equal_heads_reduces_to_plain_pull():
    nl, nb, h = 2, 9, 2
    src = _layers(nl, nb, h, 7)
    d1 = _layers(nl, nb, h, 8)
    d2 = [d.copy() for d in d1]
    s_ids, d_ids = kvdgen.random_table(5, nb, nb, seed=1)
    assert oracle.pull_heads(src, (0,) * 5, nb, h, d1, (0,) * 5, nb, h, 0, D, L, E,
                             s_ids, d_ids) == oracle.OK
    assert oracle.pull(src, (0,) * 5, nb, d2, (0,) * 5, nb, h, D, L, E, s_ids, d_ids) == oracle.OK
    for a, b in zip(d1, d2):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("off,s_ids,d_ids,rc", [
    (2, [0], [0], oracle.EINVAL),          # heads 2..3 do not fit in 3 destination heads
    (0, [0, 12], [1, 2], oracle.ERANGE),
    (0, [0, 1], [2, 2], oracle.EINVAL),
])
def test_head_errors_write_nothing(off, s_ids, d_ids, rc):
    nb = 12
    src = _layers(1, nb, 2, 1)
    dst = _layers(1, nb, 3, 2)
    before = dst[0].copy()
    got = oracle.pull_heads(src, (0,) * 5, nb, 2, dst, (0,) * 5, nb, 3, off, D, L, E,
                            np.array(s_ids, np.int32), np.array(d_ids, np.int32))
    assert got == rc
    assert np.array_equal(before, dst[0])
