#!/usr/bin/env python
"""C5 transfer sweep (BASELINE.json configs[4]): block size 8/16/32 x run
length 1..64 blocks x model {7B, 70B-TP4 shard}, 8K-token requests, at
N = 2/4/8 GPUs (N/2 concurrent rail pairs), pull (coalescing on and off)
vs the NCCL N1 send/recv baseline on the same caches and block tables.

    torchrun --nproc-per-node N tools/c5_sweep.py [--iters 10] [--models 7b,70b]

One JSON line per point on rank 0.  Pull GB/s = bytes per pair / device time
(CUDA events around the launch), aggregated as the sum over pairs / max time;
NCCL = host wall per request (incl. the block-id message), max over ranks:
N1 (whole request staged), N3 (double-buffered chunks, chunk size swept)
and N0 (one contiguous message of the same bytes, NCCL's link ceiling);
the pull is compared with the best paged-transfer variant.  Every point is
parity-checked element by element (bench.decode_matches: the decode cache
equals its regenerated pre-state with the pulled blocks replaced by the
regenerated source blocks).
"""
import argparse
import json
import os
import sys
import time
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch
import torch.distributed as dist

import bench
import kvdgen
from paper_2501_14743_b200 import cluster, kvd
from paper_2501_14743_b200.torch_cache import PagedCache

MODELS = {"7b": (32, 32, 128, kvdgen.FP16), "70b": (80, 2, 128, kvdgen.BF16)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--models", default="7b,70b")
    ap.add_argument("--bs", default="8,16,32")
    ap.add_argument("--runs", default="1,2,4,8,16,32,64")
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--variant", default="", help="force lsu|lsu32|tma (default: library auto)")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    gloo = dist.new_group(backend="gloo")
    me = cluster.role_of(rank, world)
    half = world // 2
    stream = torch.cuda.Stream(dev)
    rid = [rank * 10_000_000]
    for model in a.models.split(","):
        NL, H, D, dt = MODELS[model]
        for bs in [int(x) for x in a.bs.split(",")]:
            for r in [int(x) for x in a.runs.split(",")]:
                n = a.tokens // bs
                nb = n + n // r + 16
                g = kvdgen.CacheGeom(NL, H, D, bs, nb, dt)
                s_ids, d_ids = kvdgen.fixed_run_table(n, r, nb, nb, seed=bs * 100 + r)
                cache = PagedCache(NL, H, D, bs, nb, dt, (0,) * 5, dev)
                for l, t in enumerate(cache.layers):
                    kvdgen.torch_fill_random_(t, rank * 1000 + l)
                torch.cuda.synchronize()
                src = cache if me.role == "prefill" else None
                dst = cache if me.role == "decode" else None
                blob = cluster.peer_blob(me, cluster.exchange_blobs(src.export() if src else None, gloo))
                peer = dst.open_peer(blob) if dst else None
                if peer and a.variant:
                    peer.set(kvd.OPT_VARIANT, {"lsu": 1, "lsu32": 2, "tma": 4}[a.variant])
                res = {}
                for label, coalesce in (("pull", 1), ("pull_nocoalesce", 0)):
                    t_dev = 0.0
                    if peer:
                        peer.set(kvd.OPT_COALESCE, coalesce)
                        for _ in range(2):
                            rid[0] += 1
                            peer.pull(rid[0], s_ids, d_ids, stream)
                            peer.wait(rid[0])
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        dist.barrier(group=gloo)
                        e0.record(stream)
                        for _ in range(a.iters):
                            rid[0] += 1
                            peer.pull(rid[0], s_ids, d_ids, stream)
                            peer.wait(rid[0])
                        e1.record(stream)
                        torch.cuda.synchronize()
                        t_dev = e0.elapsed_time(e1) / 1e3
                        info = peer.info()
                    else:
                        dist.barrier(group=gloo)
                        info = {}
                    res[label] = {"t": t_dev, "runs": info.get("runs"), "variant": info.get("variant"),
                                  "ctas": info.get("ctas"), "threads": info.get("threads")}
                span = cache.span_bytes
                per = n * NL * 2 * span
                # caches were filled with seed rank * 1000 + l: the source is
                # the prefill rank's, the pre-state this rank's
                ok = (bench.decode_matches(dst, g, s_ids, d_ids, me.peer, rank, dev)
                      if dst else True)
                base = {}
                if not a.no_nccl:
                    args = types.SimpleNamespace(steps=a.iters, no_n2=True)
                    base = bench.nccl_baselines(args, g, [(s_ids, d_ids)], src, dst, me.role, rank, half,
                                                dev, gloo, me.peer)
                stats = {"res": res, "ok": ok, "base": base, "bytes": per if dst else 0}
                all_s = cluster.gather_stats(stats, gloo)
                if rank == 0:
                    dec = [s for s in all_s if s["bytes"]]
                    pairs = len(dec)
                    out = {"model": model, "block_size": bs, "run_blocks": r, "blocks": n,
                           "bytes_per_pair": per, "span_bytes": span, "pairs": pairs, "n_gpus": world}
                    for label in ("pull", "pull_nocoalesce"):
                        t = max(s["res"][label]["t"] for s in dec)
                        out[label + "_gbs_per_pair"] = round(per * a.iters / t / 1e9, 1)
                        out[label + "_runs"] = dec[0]["res"][label]["runs"]
                    out["variant"] = dec[0]["res"]["pull"]["variant"]
                    out["threads"] = dec[0]["res"]["pull"].get("threads")
                    out["ctas"] = dec[0]["res"]["pull"]["ctas"]
                    if not a.no_nccl:
                        nccl = {}
                        for name in dec[0]["base"]:
                            rs = [s["base"][name] for s in dec]
                            t = max(x["wall_s"] for x in rs)
                            nccl[name] = round(per * rs[0]["steps"] / t / 1e9, 1)
                        out["nccl_gbs_per_pair"] = nccl
                        out["nccl_parity"] = all(v["ok"] for s in all_s if s["base"]
                                                 for v in s["base"].values())
                        transfers = {k: v for k, v in nccl.items() if not k.startswith("n0")}
                        best = max(transfers, key=transfers.get)
                        out["nccl_best_transfer"] = best
                        out["pull_vs_best_nccl"] = round(out["pull_gbs_per_pair"] / transfers[best], 2)
                        out["pull_vs_nccl_n0_ceiling"] = round(
                            out["pull_gbs_per_pair"] / nccl["n0_raw_contiguous"], 2)
                    out["parity"] = all(s["ok"] for s in all_s)
                    print(json.dumps(out), flush=True)
                if peer:
                    peer.close()
                dist.barrier(group=gloo)
                cache.close()
                del cache
                torch.cuda.empty_cache()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
