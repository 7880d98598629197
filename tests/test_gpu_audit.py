"""Bounds audit (KVD_OPT_AUDIT): compute-sanitizer is closed on this pool, so
every mover checks in-kernel that each tile it copies stays inside its layer
tensors on both sides.  Here every path -- LSU / LSU32 / TMA / small-request,
the resident engine, single and batched pulls, push, head slices, padded and
folded layouts, ragged
tiles -- runs with the audit on: zero violations, and the bytes still match
the oracle."""
import numpy as np
import pytest
import torch

import kvdgen
from gpu_helpers import assert_layers_equal, make_pair, next_request_id, pull_and_wait
from paper_2501_14743_b200 import kvd

pytestmark = pytest.mark.gpu

SUB = 16 * 2 * 64
LAYOUTS = [(0,) * 5, (2 * SUB, SUB, 128, 64, 1), (3 * SUB, SUB, 128, 64, 1)]
CFGS = [
    {},
    {kvd.OPT_VARIANT: kvd.VARIANT_LSU, kvd.OPT_TILE_BYTES: 1536 // 512 * 512},
    {kvd.OPT_VARIANT: kvd.VARIANT_LSU32, kvd.OPT_TILE_BYTES: 4096},
    {kvd.OPT_VARIANT: kvd.VARIANT_TMA, kvd.OPT_TILE_BYTES: 3072, kvd.OPT_STAGES: 3,
     kvd.OPT_THREADS: 64},
    {kvd.OPT_VARIANT: kvd.VARIANT_TMA, kvd.OPT_TILE_BYTES: 16384, kvd.OPT_STAGES: 2},
    {kvd.OPT_ENGINE: 4},          # single pulls posted to the resident engine
]


@pytest.mark.parametrize("stride", LAYOUTS)
@pytest.mark.parametrize("cfg", range(len(CFGS)))
def test_audit_single_and_batched(stride, cfg):
    g = kvdgen.CacheGeom(2, 2, 64, 16, 64, kvdgen.FP16, stride)
    pair = make_pair(g, g, seed=40 + cfg)
    try:
        pair.peer.set(kvd.OPT_AUDIT, 1)
        for k, v in CFGS[cfg].items():
            pair.peer.set(k, v)
        exp = pair.dst_host
        for kind in range(3):
            s, d = kvdgen.random_table(20 + kind, 64, 64, seed=kind)
            pull_and_wait(pair, s, d)
            exp = pair.expected(s, d, exp)
        tables = kvdgen.disjoint_fragmented_tables([5, 0, 9, 13], 64, 64, seed=cfg)
        rids = [next_request_id() for _ in tables]
        pair.peer.pull_batch(rids, tables)
        for r in rids:
            pair.peer.wait(r)
        for s, d in tables:
            exp = pair.expected(s, d, exp)
        assert pair.peer.audit() == 0
        assert_layers_equal(pair.download_dst(), exp)
    finally:
        pair.close()


def test_audit_push_and_heads():
    g = kvdgen.CacheGeom(3, 2, 64, 16, 64, kvdgen.BF16)
    pair = make_pair(g, g, seed=50)
    try:
        rev = pair.src.open_peer(pair.dst.export())
        rev.set(kvd.OPT_AUDIT, 1)
        s, d = kvdgen.fragmented_table(30, 64, 64, seed=1)
        rid = next_request_id()
        rev.push(rid, s, d)
        rev.wait(rid)
        assert rev.audit() == 0
        assert_layers_equal(pair.download_dst(), pair.expected(s, d))
        rev.close()
    finally:
        pair.close()
    from gpu_helpers import cache_for
    shard = cache_for(kvdgen.CacheGeom(2, 1, 128, 16, 32, kvdgen.BF16), 0)
    dst = cache_for(kvdgen.CacheGeom(2, 4, 128, 16, 32, kvdgen.BF16), 0)
    try:
        p = dst.open_peer_heads(shard.export(), 3)           # the last head slot
        p.set(kvd.OPT_AUDIT, 1)
        rid = next_request_id()
        p.pull(rid, np.arange(10, dtype=np.int32), np.arange(22, 32, dtype=np.int32))
        p.wait(rid)
        assert p.audit() == 0
        p.close()
    finally:
        dst.close()
        shard.close()


def test_audit_off_reports_state_error():
    pair = make_pair(kvdgen.C1, kvdgen.C1, seed=51)
    try:
        with pytest.raises(kvd.KvdError) as ei:
            pair.peer.audit()
        assert ei.value.status == kvd.ESTATE
    finally:
        pair.close()
