#!/usr/bin/env python
"""Per-request latency breakdown for small pulls (C1) -- where do the
microseconds go?  host call (kvd_pull), call-return -> done (poll), total."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import kvdgen
from paper_2501_14743_b200 import kvd
from paper_2501_14743_b200.torch_cache import PagedCache


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--src-dev", type=int, default=0)
    ap.add_argument("--dst-dev", type=int, default=1)
    ap.add_argument("--iters", type=int, default=2000)
    a = ap.parse_args()
    g = kvdgen.C1
    n = 16
    src = PagedCache(g.num_layers, g.num_kv_heads, g.head_dim, g.block_size, g.num_blocks, g.dtype,
                     g.stride, a.src_dev)
    dst = PagedCache(g.num_layers, g.num_kv_heads, g.head_dim, g.block_size, g.num_blocks, g.dtype,
                     g.stride, a.dst_dev)
    torch.cuda.synchronize()
    tables = {"fragmented": kvdgen.fragmented_table(n, 64, 64, seed=0),
              "contiguous": kvdgen.contiguous_table(n, 0, 48),
              "empty": (np.zeros(0, np.int32), np.zeros(0, np.int32))}
    configs = [("auto", {}), ("lsu", {kvd.OPT_VARIANT: 1}),
               ("lsu_t128_tile4k", {kvd.OPT_VARIANT: 1, kvd.OPT_THREADS: 128,
                                    kvd.OPT_TILE_BYTES: 4096}),
               ("tma_tile8k", {kvd.OPT_VARIANT: 4, kvd.OPT_THREADS: 32, kvd.OPT_TILE_BYTES: 8192}),
               ("tma_tile4k_s2", {kvd.OPT_VARIANT: 4, kvd.OPT_THREADS: 32, kvd.OPT_TILE_BYTES: 4096,
                                  kvd.OPT_STAGES: 2}),
               ("lsu_t32_tile4k", {kvd.OPT_VARIANT: 1, kvd.OPT_THREADS: 32, kvd.OPT_TILE_BYTES: 4096}),
               ("lsu_t32_tile2k", {kvd.OPT_VARIANT: 1, kvd.OPT_THREADS: 32, kvd.OPT_TILE_BYTES: 2048}),
               ("lsu_t64_tile4k", {kvd.OPT_VARIANT: 1, kvd.OPT_THREADS: 64, kvd.OPT_TILE_BYTES: 4096})]
    stream = torch.cuda.Stream(a.dst_dev)
    rid = 0
    # ctypes + validation floor: the host-only planner on the same table
    s, d = tables["fragmented"]
    t = []
    for _ in range(2000):
        t0 = time.perf_counter_ns()
        kvd.kvd_plan(s, d, 64, 64)
        t.append(time.perf_counter_ns() - t0)
    print(json.dumps({"kvd_plan_call_us_p50": np.median(t) / 1e3}), flush=True)
    for cname, opts in configs:
        peer = dst.open_peer(src.export())
        h = peer.handle
        for k, v in opts.items():
            kvd.kvd_peer_set(h, k, v)
        for tname, (s, d) in tables.items():
            s = np.ascontiguousarray(s, np.int32)
            d = np.ascontiguousarray(d, np.int32)
            call, rest, tot = [], [], []
            for it in range(a.iters + 50):
                rid += 1
                t0 = time.perf_counter_ns()
                kvd.kvd_pull(h, rid, s, d, stream.cuda_stream)
                t1 = time.perf_counter_ns()
                kvd.kvd_wait_done(h, rid, 10_000_000)
                t2 = time.perf_counter_ns()
                if it >= 50:
                    call.append(t1 - t0); rest.append(t2 - t1); tot.append(t2 - t0)
            info = kvd.kvd_last_pull_info(h).as_dict()
            print(json.dumps({"config": cname, "table": tname, "ctas": info["ctas"],
                              "threads": info["threads"], "tiles": info["tiles"],
                              "variant": info["variant"],
                              "call_us_p50": np.median(call) / 1e3,
                              "to_done_us_p50": np.median(rest) / 1e3,
                              "total_us_p50": np.median(tot) / 1e3,
                              "total_us_p90": float(np.percentile(tot, 90)) / 1e3}), flush=True)
        peer.close()


if __name__ == "__main__":
    main()
