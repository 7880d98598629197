#!/usr/bin/env python
"""Many short requests over one pair: back-to-back kvd_pull calls vs one
kvd_pull_batch (§8 f1) for the same block tables.  Short prompts on a 70B TP
shard move little per request, so the fixed per-request cost (launch,
completion) dominates unless the queue is drained in one
launch.  Single process, caches on --src-dev / --dst-dev.

    python tools/small_requests.py --config c4 --tokens 256,1024,4096 --requests 32
"""
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
from paper_2501_14743_b200.torch_cache import PagedCache


def _exporter(conn, dev, geom):
    """--ipc: the prefill cache lives in another process (the deployment
    shape): fill it, export the blob, keep it alive until told to stop."""
    sys.path.insert(0, ROOT)
    import torch
    torch.cuda.set_device(dev)
    g = geom
    src = PagedCache(g.num_layers, g.num_kv_heads, g.head_dim, g.block_size, g.num_blocks,
                     g.dtype, g.stride, dev)
    for l in range(g.num_layers):
        kvdgen.torch_fill_random_(src.layers[l], 10 + l)
    torch.cuda.synchronize(dev)
    conn.send((src.export(), src.span_bytes))
    conn.recv()
    src.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--src-dev", type=int, default=0)
    ap.add_argument("--dst-dev", type=int, default=1)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--tokens", default="256,1024,4096")
    ap.add_argument("--requests", type=int, default=32)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--variant", type=int, default=0, help="force a mover (kvd.VARIANT_*)")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--modes", default="single,batch,merged")
    ap.add_argument("--timing", type=int, default=2, choices=(0, 1, 2),
                    help="KVD_OPT_TIMING: 2 (default) in-kernel %%globaltimer spans only; 1 also "
                         "library events around every launch (they break PDL adjacency); 0 off")
    ap.add_argument("--early", type=int, default=2,
                    help="KVD_OPT_EARLY_LOADS (the library default, 2: the next pull's first two "
                         "ring stages of source reads overlap the previous pull's tail)")
    ap.add_argument("--ipc", action="store_true",
                    help="prefill cache in a second process (CUDA IPC mapping, as deployed)")
    a = ap.parse_args()
    base = {"c2": kvdgen.C2, "c4": kvdgen.C4}[a.config]
    toks = [int(t) for t in a.tokens.split(",")]
    need = max(kvdgen.blocks_for(t, base.block_size) for t in toks) * a.requests
    # pools ~20 % larger than the blocks in use (C3's occupancy): a nearly
    # full pool would leave no room for the gaps of a fragmented placement
    g = base.with_blocks(max(need * 6 // 5 + 64, 256))
    mk = lambda dev: PagedCache(g.num_layers, g.num_kv_heads, g.head_dim, g.block_size,
                                g.num_blocks, g.dtype, g.stride, dev)
    child = None
    if a.ipc:
        import multiprocessing as mp
        ctx = mp.get_context("spawn")
        conn, cconn = ctx.Pipe()
        child = ctx.Process(target=_exporter, args=(cconn, a.src_dev, g))
        child.start()
        blob, span = conn.recv()
        src = None
    else:
        src = mk(a.src_dev)
        for l in range(g.num_layers):
            kvdgen.torch_fill_random_(src.layers[l], 10 + l)
        torch.cuda.synchronize(a.src_dev)
        blob, span = src.export(), src.span_bytes
    dst = mk(a.dst_dev)
    peer = dst.open_peer(blob)
    from paper_2501_14743_b200 import kvd
    if a.variant:
        peer.set(kvd.OPT_VARIANT, a.variant)
    if a.threads:
        peer.set(kvd.OPT_THREADS, a.threads)
    if a.stages:
        peer.set(kvd.OPT_STAGES, a.stages)
    if a.ctas:
        peer.set(kvd.OPT_MAX_CTAS, a.ctas)
    peer.set(kvd.OPT_EARLY_LOADS, a.early)
    if a.timing:
        peer.set(kvd.OPT_TIMING, a.timing)   # in-kernel %globaltimer spans of single pulls
    torch.cuda.set_device(a.dst_dev)
    stream = torch.cuda.Stream(a.dst_dev)
    stream2 = torch.cuda.Stream(a.dst_dev)
    rid = [0]
    for t in toks:
        n = kvdgen.blocks_for(t, g.block_size)
        tables = kvdgen.disjoint_fragmented_tables([n] * a.requests, g.num_blocks, g.num_blocks,
                                                   seed=t)
        nbytes = n * a.requests * g.num_layers * 2 * span
        res = {"config": a.config, "ipc": a.ipc, "tokens_per_request": t, "requests": a.requests,
               "bytes": nbytes, "opts": {"variant": a.variant, "threads": a.threads,
                                         "stages": a.stages, "ctas": a.ctas, "early": a.early}}
        merged = (np.concatenate([s for s, _ in tables]), np.concatenate([d for _, d in tables]))
        for mode in a.modes.split(","):
            times = []
            for it in range(a.iters + 2):
                ids = []
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(stream):
                    torch.cuda._sleep(2_000_000)       # host issue hidden behind ~1 ms
                e0.record(stream)
                if mode == "single":
                    for s, d in tables:
                        rid[0] += 1
                        peer.pull(rid[0], s, d, stream)
                        ids.append(rid[0])
                elif mode == "lib2":   # KVD_OPT_STREAMS = 2: the library overlaps consecutive pulls
                    peer.set(kvd.OPT_STREAMS, 2)
                    for s, d in tables:
                        rid[0] += 1
                        peer.pull(rid[0], s, d, stream)
                        ids.append(rid[0])
                    peer.stream_wait(stream)
                elif mode == "single2":   # alternate two streams: consecutive pulls may overlap
                    stream2.wait_stream(stream)
                    for k, (s, d) in enumerate(tables):
                        rid[0] += 1
                        peer.pull(rid[0], s, d, stream if k % 2 == 0 else stream2)
                        ids.append(rid[0])
                    stream.wait_stream(stream2)
                elif mode == "batch1":   # the same blocks as a batch of ONE request
                    rid[0] += 1
                    peer.pull_batch([rid[0]], [merged], stream)
                    ids.append(rid[0])
                elif mode == "merged":   # the same blocks as ONE request: the table's own rate
                    rid[0] += 1
                    peer.pull(rid[0], merged[0], merged[1], stream)
                    ids.append(rid[0])
                else:
                    ids = list(range(rid[0] + 1, rid[0] + 1 + len(tables)))
                    rid[0] += len(tables)
                    peer.pull_batch(ids, tables, stream)
                e1.record(stream)
                for r in ids:
                    peer.wait(r)
                e1.synchronize()
                if mode == "lib2":
                    peer.set(kvd.OPT_STREAMS, 0)
                if it >= 2:
                    times.append(e0.elapsed_time(e1))
            ms = float(np.median(times))
            gt_ms, gt_n = peer.device_time()
            if a.timing == 1:
                peer.kernel_time()                 # drop the launch events
            if gt_n:   # mean in-kernel span per request vs the per-request share of the step
                res[mode + "_kernel_us_per_request"] = round(gt_ms / gt_n * 1e3, 2)
                res[mode + "_step_us_per_request"] = round(
                    ms * 1e3 / (len(tables) if mode in ("single", "single2", "lib2") else 1), 2)
            res[mode + "_ms"] = round(ms, 4)
            res[mode + "_gbs"] = round(nbytes / ms / 1e6, 1)
            res[mode + "_info"] = {k: peer.info()[k] for k in ("variant", "ctas", "threads", "runs")}
        print(json.dumps(res), flush=True)
    peer.close()
    dst.close()
    if src is not None:
        src.close()
    if child is not None:
        conn.send("done")
        child.join(60)


if __name__ == "__main__":
    main()
