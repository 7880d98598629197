#!/usr/bin/env python
"""Pull vs push when both directions of a GPU pair carry a transfer at once
(DESIGN.md §8 ring stress; the transfer-level side of the paper's pull-vs-push
comparison).  GPU0 and GPU1 each hold a "prefill" and a "decode" C2
cache; the same fragmented 8K-token request moves GPU0 -> GPU1 and GPU1 -> GPU0
concurrently, either pulled (the decode GPU's kernel reads over NVLink) or
pushed (the prefill GPU's kernel writes over NVLink), auto policy; and one
direction alone for reference.  GB/s per direction = bytes / the slower of the
two devices' CUDA-event times; parity of both decode caches is checked
against the regenerated source blocks.

    python tools/bidir_probe.py [--iters 10]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import kvdgen
from paper_2501_14743_b200.torch_cache import PagedCache


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    g = kvdgen.C2
    mk = lambda dev, seed: fill(PagedCache(g.num_layers, g.num_kv_heads, g.head_dim, g.block_size,
                                           g.num_blocks, g.dtype, g.stride, dev), seed)

    def fill(c, seed):
        for l, t in enumerate(c.layers):
            kvdgen.torch_fill_random_(t, seed * 1000 + l)
        return c

    src = [mk(0, 1), mk(1, 2)]       # prefill caches on GPU0 / GPU1
    dst = [mk(0, 3), mk(1, 4)]       # decode caches on GPU0 / GPU1
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    # pull: decode GPU d imports the other GPU's prefill cache
    pulls = [dst[d].open_peer(src[1 - d].export()) for d in (0, 1)]
    # push: prefill GPU p imports the other GPU's decode cache
    pushes = [src[p].open_peer(dst[1 - p].export()) for p in (0, 1)]
    n = kvdgen.blocks_for(kvdgen.C2_TOKENS, g.block_size)
    s_ids, d_ids = kvdgen.fragmented_table(n, g.num_blocks, g.num_blocks, seed=1)
    nbytes = n * g.num_layers * 2 * src[0].span_bytes
    streams = [torch.cuda.Stream(0), torch.cuda.Stream(1)]
    rid = [0]

    def run(peers, devs, push):
        for _ in range(2):       # warm-up
            go(peers, devs, push)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in devs]
        ids = []
        for k, d in enumerate(devs):
            with torch.cuda.device(d):
                ev[k][0].record(streams[d])
        for _ in range(a.iters):
            ids += go(peers, devs, push, wait=False)
        for k, d in enumerate(devs):
            with torch.cuda.device(d):
                ev[k][1].record(streams[d])
        for p, r in ids:
            p.wait(r)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        ms = max(e0.elapsed_time(e1) for e0, e1 in ev)
        return round(nbytes * a.iters / (ms / 1e3) / 1e9, 1)

    def go(peers, devs, push, wait=True):
        ids = []
        for d in devs:
            p = peers[d]
            rid[0] += 1
            if push:
                p.push(rid[0], s_ids, d_ids, streams[d])
            else:
                p.pull(rid[0], s_ids, d_ids, streams[d])
            ids.append((p, rid[0]))
        if wait:
            for p, r in ids:
                p.wait(r)
        return ids

    out = {"bytes_per_request": nbytes, "iters": a.iters}
    # pull: the kernel runs on the decode GPU d (pulls[d] local = dst[d]);
    # push: on the prefill GPU p (pushes[p] local = src[p])
    out["pull_one_way_gbs"] = run(pulls, [1], False)
    out["pull_both_ways_gbs_per_direction"] = run(pulls, [0, 1], False)
    out["push_one_way_gbs"] = run(pushes, [0], True)
    out["push_both_ways_gbs_per_direction"] = run(pushes, [0, 1], True)
    ok = True
    si = torch.tensor(s_ids, dtype=torch.long)
    di = torch.tensor(d_ids, dtype=torch.long)
    span = src[0].span_bytes
    for d in (0, 1):             # dst[d]'s blocks d_ids == src[1-d]'s blocks s_ids
        for l in range(g.num_layers):
            a_ = dst[d].layers[l].view(2, g.num_blocks, span)[:, di.to(f"cuda:{d}")]
            b_ = src[1 - d].layers[l].view(2, g.num_blocks, span)[:, si.to(f"cuda:{1 - d}")]
            ok = ok and bool(torch.equal(a_.cpu(), b_.cpu()))
    out["parity"] = ok
    print(json.dumps(out), flush=True)
    for p in pulls + pushes:
        p.close()


if __name__ == "__main__":
    main()
