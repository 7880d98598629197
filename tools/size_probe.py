#!/usr/bin/env python
"""Kernel time vs request size over one pair (single process, two GPUs):
fits t(n) = F + bytes / R to split the fixed per-request overhead F from the
streaming rate R, per mover / launch policy.

    python tools/size_probe.py --config c2 --variants auto,tma,lsu32 > out.jsonl
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import kvdgen
from paper_2501_14743_b200 import kvd
from paper_2501_14743_b200.torch_cache import PagedCache

VAR = {"auto": 0, "lsu": 1, "lsu32": 2, "tma": 4}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--src-dev", type=int, default=0)
    ap.add_argument("--dst-dev", type=int, default=1)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--variants", default="auto")
    ap.add_argument("--table", default="contiguous")
    ap.add_argument("--sizes", default="1,2,4,8,16,32,64,128,256,512")
    ap.add_argument("--ctas", default="0")
    ap.add_argument("--iters", type=int, default=15)
    ap.add_argument("--layers", type=int, default=0, help="override the config's layer count")
    ap.add_argument("--hide-host", type=int, default=1,
                    help="1: a ~100 us sleep kernel ahead of each pull, so the events time the "
                         "GPU work only (not the host issue gap)")
    a = ap.parse_args()
    g = {"c1": kvdgen.C1, "c2": kvdgen.C2, "c4": kvdgen.C4}[a.config]
    if a.layers:
        from dataclasses import replace
        g = replace(g, num_layers=a.layers)
    mk = lambda dev: PagedCache(g.num_layers, g.num_kv_heads, g.head_dim, g.block_size,
                                g.num_blocks, g.dtype, g.stride, dev)
    src, dst = mk(a.src_dev), mk(a.dst_dev)
    for l in range(g.num_layers):
        kvdgen.torch_fill_random_(src.layers[l], 10 + l)
    torch.cuda.synchronize(a.src_dev)
    peer = dst.open_peer(src.export())
    torch.cuda.set_device(a.dst_dev)
    stream = torch.cuda.Stream(a.dst_dev)
    rid = [0]
    for var in a.variants.split(","):
        for ctas in [int(c) for c in a.ctas.split(",")]:
            peer.set(kvd.OPT_VARIANT, VAR[var]).set(kvd.OPT_MAX_CTAS, ctas)
            pts = []
            for n in [int(x) for x in a.sizes.split(",")]:
                if a.table == "contiguous":
                    s, d = kvdgen.contiguous_table(n, 0, g.num_blocks - n)
                else:
                    s, d = kvdgen.fragmented_table(n, g.num_blocks, g.num_blocks, seed=1)
                ms = []
                for k in range(a.iters + 3):
                    e0, e1 = (torch.cuda.Event(enable_timing=True),
                              torch.cuda.Event(enable_timing=True))
                    rid[0] += 1
                    if a.hide_host:   # keep the stream busy while the host issues the pull
                        with torch.cuda.stream(stream):
                            torch.cuda._sleep(200_000)
                    e0.record(stream)
                    peer.pull(rid[0], s, d, stream)
                    e1.record(stream)
                    peer.wait(rid[0])
                    e1.synchronize()
                    if k >= 3:
                        ms.append(e0.elapsed_time(e1))
                info = peer.info()
                t = float(np.median(ms))
                pts.append((info["bytes"], t))
                print(json.dumps({"config": a.config, "variant": var, "table": a.table,
                                  "hide_host": a.hide_host,
                                  "blocks": n, "bytes": info["bytes"], "ctas": info["ctas"],
                                  "threads": info["threads"], "mover": info["variant"],
                                  "ms": round(t, 4),
                                  "gbs": round(info["bytes"] / t / 1e6, 1) if n else 0.0}),
                      flush=True)
            if len(pts) < 3:
                continue
            b = np.array([p[0] for p in pts], float)
            t = np.array([p[1] for p in pts], float)
            big = b >= b.max() / 16
            A = np.vstack([np.ones(big.sum()), b[big]]).T
            (F, inv), *_ = np.linalg.lstsq(A, t[big], rcond=None)
            print(json.dumps({"fit": True, "config": a.config, "variant": var, "ctas": ctas,
                              "hide_host": a.hide_host,
                              "table": a.table, "fixed_us": round(F * 1e3, 2),
                              "rate_gbs": round(1 / inv / 1e6, 1)}), flush=True)
    peer.close()
    dst.close()
    src.close()


if __name__ == "__main__":
    main()
