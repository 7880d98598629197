#!/usr/bin/env python
"""Small single-GPU workload for compute-sanitizer (one tool per run):
every mover (LSU, LSU32, TMA ring, small-request path), the batched drain,
the push variant and the baseline gather/scatter on C1-sized caches, each
checked against the CPU oracle.  Exit code 0 = all bit-exact."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np
import torch

import kvdgen
from gpu_helpers import assert_layers_equal, make_pair, next_request_id, pull_and_wait
from paper_2501_14743_b200 import kvd


def main():
    g = kvdgen.CacheGeom(2, 2, 64, 16, 64, kvdgen.FP16)
    pair = make_pair(g, g, seed=1)
    exp = pair.dst_host
    cfgs = [{}, {kvd.OPT_VARIANT: kvd.VARIANT_LSU, kvd.OPT_THREADS: 256},
            {kvd.OPT_VARIANT: kvd.VARIANT_LSU32},
            {kvd.OPT_VARIANT: kvd.VARIANT_TMA, kvd.OPT_TILE_BYTES: 4096, kvd.OPT_STAGES: 3}]
    for i, cfg in enumerate(cfgs):
        for k, v in cfg.items():
            pair.peer.set(k, v)
        s, d = kvdgen.random_table(16, 64, 64, seed=i)
        pull_and_wait(pair, s, d)
        exp = pair.expected(s, d, exp)
        assert_layers_equal(pair.download_dst(), exp)
    pair.peer.set(kvd.OPT_VARIANT, kvd.VARIANT_AUTO)
    tables = kvdgen.disjoint_fragmented_tables([5, 0, 9, 3], 64, 64, seed=7)
    rids = [next_request_id() for _ in tables]
    pair.peer.pull_batch(rids, tables)
    for r in rids:
        pair.peer.wait(r)
    for s, d in tables:
        exp = pair.expected(s, d, exp)
    assert_layers_equal(pair.download_dst(), exp)
    rev = pair.src.open_peer(pair.dst.export())
    s, d = kvdgen.random_table(12, 64, 64, seed=11)
    rid = next_request_id()
    rev.push(rid, s, d)
    rev.wait(rid)
    exp = pair.expected(s, d, exp)
    assert_layers_equal(pair.download_dst(), exp)
    rev.close()
    # baseline gather + scatter round trip
    ids = np.array([3, 9, 4, 60], np.int32)
    span = pair.src.span_bytes
    staging = torch.empty(2 * 2 * len(ids) * span, dtype=torch.uint8, device="cuda:0")
    kvd.kvd_gather(pair.src.handle, ids, staging.data_ptr(), torch.cuda.current_stream().cuda_stream)
    to = np.array([1, 2, 5, 7], np.int32)
    kvd.kvd_scatter(pair.dst.handle, to, staging.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    exp = pair.expected(ids, to, exp)
    assert_layers_equal(pair.download_dst(), exp)
    pair.close()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
