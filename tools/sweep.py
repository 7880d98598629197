#!/usr/bin/env python
"""Single-process pull sweeps for tuning (not the bench contract).

Caches live on --src-dev (prefill) and --dst-dev (decode) of ONE process;
with two GPUs the pull crosses NVLink exactly as in the multi-process case
(same kernel, peer mapping via cudaDeviceEnablePeerAccess instead of IPC).
Prints one JSON line per configuration: kernel GB/s from CUDA events.
Also measures the copy-engine ceiling (torch peer copy of one contiguous
buffer = cudaMemcpyPeerAsync) as a context number.
"""
import argparse
import itertools
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

VAR = {"lsu": 1, "lsu32": 2, "ce": 3, "tma": 4}


def geom_of(name):
    return {"c1": kvdgen.C1, "c2": kvdgen.C2, "c4": kvdgen.C4}[name]


def tables(g, kind, n):
    if kind == "contiguous":
        return kvdgen.contiguous_table(n, 0, g.num_blocks - n)
    if kind == "worst":
        return kvdgen.fixed_run_table(n, 1, g.num_blocks, g.num_blocks, seed=1)
    if kind.startswith("run"):
        return kvdgen.fixed_run_table(n, int(kind[3:]), g.num_blocks, g.num_blocks, seed=1)
    return kvdgen.fragmented_table(n, g.num_blocks, g.num_blocks, seed=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--src-dev", type=int, default=0)
    ap.add_argument("--dst-dev", type=int, default=1)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--block-size", type=int, default=0, help="override the config's block size")
    ap.add_argument("--tables", default="fragmented")
    ap.add_argument("--variants", default="lsu")
    ap.add_argument("--tiles", default="16384")
    ap.add_argument("--threads", default="512")
    ap.add_argument("--ctas", default="0")
    ap.add_argument("--stages", default="4")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--ce-ceiling", action="store_true")
    ap.add_argument("--mode", choices=["pull", "push"], default="pull")
    ap.add_argument("--profile-once", action="store_true",
                    help="one warm-up pull then exactly one pull (for ncu -s/-c)")
    a = ap.parse_args()
    g = geom_of(a.config)
    if a.block_size:
        from dataclasses import replace
        g = replace(g, block_size=a.block_size, num_blocks=g.num_blocks * g.block_size // a.block_size)
    n = kvdgen.blocks_for({"c1": 256, "c2": 8192, "c4": 8192}[a.config], g.block_size)
    mk = lambda dev, seed: PagedCache(g.num_layers, g.num_kv_heads, g.head_dim, g.block_size,
                                      g.num_blocks, g.dtype, g.stride, dev)
    src = mk(a.src_dev, 1)
    dst = mk(a.dst_dev, 2)
    for l in range(g.num_layers):
        kvdgen.torch_fill_random_(src.layers[l], 10 + l)
        kvdgen.torch_fill_random_(dst.layers[l], 20 + l)
    torch.cuda.synchronize(a.src_dev)
    torch.cuda.synchronize(a.dst_dev)
    if a.mode == "push":     # kernel on the prefill GPU, stores over NVLink
        peer = src.open_peer(dst.export())
        run_dev = a.src_dev
    else:
        peer = dst.open_peer(src.export())
        run_dev = a.dst_dev
    torch.cuda.set_device(run_dev)
    stream = torch.cuda.Stream(run_dev)
    go = peer.push if a.mode == "push" else peer.pull
    rid = [0]

    def pull(s, d):
        rid[0] += 1
        go(rid[0], s, d, stream)
        peer.wait(rid[0])

    if a.profile_once:
        s, d = tables(g, a.tables.split(",")[0], n)
        if a.variants != "auto":     # "auto": the library's own launch policy (bench default)
            peer.set(kvd.OPT_VARIANT, VAR[a.variants.split(",")[0]])
            peer.set(kvd.OPT_TILE_BYTES, int(a.tiles.split(",")[0]))
            peer.set(kvd.OPT_THREADS, int(a.threads.split(",")[0]))
            peer.set(kvd.OPT_MAX_CTAS, int(a.ctas.split(",")[0]))
        pull(s, d)
        torch.cuda.synchronize()
        pull(s, d)
        torch.cuda.synchronize()
        print(json.dumps({"profiled": peer.info()}))
        return

    if a.ce_ceiling:
        nbytes = 4 << 30
        x = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{a.src_dev}")
        y = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{a.dst_dev}")
        with torch.cuda.stream(stream):
            for _ in range(3):
                y.copy_(x, non_blocking=True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(5):
                y.copy_(x, non_blocking=True)
            e1.record(stream)
        torch.cuda.synchronize()
        print(json.dumps({"ce_peer_copy_gbs": round(5 * nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9, 1),
                          "bytes": nbytes, "src": a.src_dev, "dst": a.dst_dev}), flush=True)
        del x, y

    for kind, var, tile, thr, ctas, st in itertools.product(
            a.tables.split(","), a.variants.split(","), [int(t) for t in a.tiles.split(",")],
            [int(t) for t in a.threads.split(",")], [int(c) for c in a.ctas.split(",")],
            [int(x) for x in a.stages.split(",")]):
        s, d = tables(g, kind, n)
        if var == "tma" and (thr // 32) * st * tile > 225 * 1024:
            continue
        if var == "auto":   # the library's own policy (run auto before explicit shapes)
            peer.set(kvd.OPT_VARIANT, kvd.VARIANT_AUTO)
        else:
            peer.set(kvd.OPT_VARIANT, VAR[var]).set(kvd.OPT_TILE_BYTES, tile)
            peer.set(kvd.OPT_THREADS, thr).set(kvd.OPT_MAX_CTAS, ctas).set(kvd.OPT_STAGES, st)
        for _ in range(a.warmup):
            pull(s, d)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(a.iters)]
        lat = []
        for k in range(a.iters):
            ev[k][0].record(stream)
            rid[0] += 1
            t0 = time.perf_counter()
            go(rid[0], s, d, stream)
            ev[k][1].record(stream)
            peer.wait(rid[0])
            lat.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
        ms = [x.elapsed_time(y) for x, y in ev]
        info = peer.info()
        print(json.dumps({"mode": a.mode, "config": a.config, "table": kind, "variant": var, "tile": tile,
                          "threads": thr, "stages": st, "ctas": info["ctas"], "runs": info["runs"],
                          "kernel_ms_med": round(float(np.median(ms)), 4),
                          "gbs": round(info["bytes"] / (np.median(ms) / 1e3) / 1e9, 1),
                          "p50_lat_ms": round(float(np.median(lat)) * 1e3, 4)}), flush=True)
    peer.close(); dst.close(); src.close()


if __name__ == "__main__":
    main()
