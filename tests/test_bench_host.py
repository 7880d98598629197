"""bench.py's host logic on CPU: the workload each pair pulls (BASELINE.json
configs, SURVEY.md §8 d), the nearest-rank percentile, and the pairing at
every N the scaling run uses (1, 2, 4, 8)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import kvdgen  # noqa: E402
from paper_2501_14743_b200 import cluster, kvd  # noqa: E402


def test_nearest_rank_percentile():
    xs = [5, 1, 4, 2, 3]
    assert bench.nearest_rank(xs, 50) == 3
    assert bench.nearest_rank(xs, 90) == 5
    assert bench.nearest_rank(xs, 0) == 1
    assert bench.nearest_rank(xs, 100) == 5
    assert bench.nearest_rank([], 50) is None
    assert bench.nearest_rank(list(range(1, 101)), 50) == 50


@pytest.mark.parametrize("config,blocks,layers", [("c1", 16, 2), ("c2", 512, 32), ("c4", 512, 80)])
def test_single_request_workloads(config, blocks, layers):
    g, reqs, desc = bench.workload(config, "fragmented")
    assert len(reqs) == 1 and len(reqs[0][0]) == blocks and g.num_layers == layers
    s, d = reqs[0]
    assert len(set(d.tolist())) == blocks                     # distinct destinations
    assert 0 <= s.min() and s.max() < g.num_blocks and d.max() < g.num_blocks
    if config == "c2":                                      # the bench's 130-run table
        assert len(kvd.kvd_plan(s, d, g.num_blocks, g.num_blocks)) == 130


def test_c3_partition_over_four_pairs():
    """C3: request i goes to pair i % 4; the four pairs together pull all 64
    requests (307,167 tokens), each into disjoint destination blocks."""
    toks = kvdgen.mixed_request_tokens(kvdgen.C3_REQUESTS, seed=0)
    assert len(toks) == 64 and sum(toks) == 307167
    total_blocks = 0
    for k in range(4):
        g, reqs, _ = bench.workload("c3", "fragmented", pair_index=k)
        mine = [t for i, t in enumerate(toks) if i % 4 == k]
        assert [len(s) for s, _ in reqs] == [kvdgen.blocks_for(t, 16) for t in mine]
        dst = np.concatenate([d for _, d in reqs])
        assert len(set(dst.tolist())) == len(dst)               # disjoint within the pair
        total_blocks += len(dst)
    assert total_blocks == sum(kvdgen.blocks_for(t, 16) for t in toks) == 19227


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_pairing_at_every_scaling_point(world):
    roles = [cluster.role_of(r, world) for r in range(world)]
    if world == 1:
        assert roles[0].role == "both"
        return
    half = world // 2
    assert [r.role for r in roles] == ["prefill"] * half + ["decode"] * half
    for r in roles:                                         # rail rule: k <-> half + k
        assert roles[r.peer].peer == r.rank and abs(r.peer - r.rank) == half
        assert r.pairs == half


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_ring_pairing(world):
    """bench.py --pairing ring: every rank holds both caches and pulls from
    its successor, so each rank is pulled from exactly once."""
    roles = [cluster.ring_role_of(r, world) for r in range(world)]
    assert all(r.role == "both" for r in roles)
    if world > 1:
        assert sorted(r.peer for r in roles) == list(range(world))
        assert all(r.peer != r.rank for r in roles)
        blobs = [f"blob{r}".encode() for r in range(world)]
        assert [cluster.peer_blob(r, blobs) for r in roles] == \
               [blobs[(r + 1) % world] for r in range(world)]
