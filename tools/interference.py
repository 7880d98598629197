#!/usr/bin/env python
"""How much does a pull disturb decode compute on the decode GPU (and vice
versa)?  A bf16 GEMM loop (stand-in for decode work) runs on one stream while
C2 pulls run on another; both throughputs are measured alone and overlapped
for each mover: TMA ring (32 SMs), LSU (all SMs), copy engine (no SMs).
Single process, GPU0 = prefill, GPU1 = decode."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import kvdgen
from paper_2501_14743_b200 import kvd
from paper_2501_14743_b200.torch_cache import PagedCache


def main():
    g = kvdgen.C2
    n = 512
    src = PagedCache(g.num_layers, g.num_kv_heads, g.head_dim, g.block_size, g.num_blocks, g.dtype, g.stride, 0)
    dst = PagedCache(g.num_layers, g.num_kv_heads, g.head_dim, g.block_size, g.num_blocks, g.dtype, g.stride, 1)
    torch.cuda.synchronize(0)
    peer = dst.open_peer(src.export())
    torch.cuda.set_device(1)
    s_ids, d_ids = kvdgen.fragmented_table(n, g.num_blocks, g.num_blocks, seed=1)
    # the copy engine issues one cudaMemcpyAsync per segment: give it the
    # contiguous table (64 segments) so it is not host-issue-bound
    c_s, c_d = kvdgen.contiguous_table(n, 0, g.num_blocks - n)
    bytes_per = n * g.num_layers * 2 * src.span_bytes
    M = 8192
    A = torch.randn(M, M, device="cuda:1", dtype=torch.bfloat16)
    B = torch.randn(M, M, device="cuda:1", dtype=torch.bfloat16)
    gemm_stream, pull_stream = torch.cuda.Stream(1), torch.cuda.Stream(1)
    rid = [0]

    def gemms(k):
        with torch.cuda.stream(gemm_stream):
            for _ in range(k):
                torch.matmul(A, B)

    table = [s_ids, d_ids]

    def pulls(k):
        for _ in range(k):
            rid[0] += 1
            peer.pull(rid[0], table[0], table[1], pull_stream)

    def timed(fn_gemm, fn_pull):
        torch.cuda.synchronize(1)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(gemm_stream)
        if fn_gemm: fn_gemm()
        g1.record(gemm_stream)
        p0.record(pull_stream)
        if fn_pull: fn_pull()
        p1.record(pull_stream)
        torch.cuda.synchronize(1)
        while True:   # retire completion slots
            try:
                for r in range(rid[0] - 64, rid[0] + 1):
                    if r > 0:
                        peer.poll(r)
            except kvd.KvdError:
                pass
            break
        return g0.elapsed_time(g1) / 1e3, p0.elapsed_time(p1) / 1e3

    KG, KP = 180, 20          # ~120 ms of GEMMs against ~110 ms of pulls
    flop = 2 * M ** 3
    gemms(5); torch.cuda.synchronize(1)
    tg, _ = timed(lambda: gemms(KG), None)
    base_tflops = KG * flop / tg / 1e12
    out = {"gemm_alone_tflops": round(base_tflops, 1)}
    tma_ctas = [int(x) for x in os.environ.get("TMA_CTAS", "32").split(",")]
    cfgs = [(f"tma{c}" if len(tma_ctas) > 1 else "tma",
             {kvd.OPT_VARIANT: kvd.VARIANT_TMA, kvd.OPT_THREADS: 32, kvd.OPT_STAGES: 6,
              kvd.OPT_TILE_BYTES: 32768, kvd.OPT_MAX_CTAS: c}) for c in tma_ctas]
    # "auto" first: the library's own launch policy (later configs set
    # options that stay set on the peer)
    for name, opts in (("auto", {}), *cfgs,
                       ("lsu", {kvd.OPT_VARIANT: kvd.VARIANT_LSU32, kvd.OPT_THREADS: 512,
                                kvd.OPT_TILE_BYTES: 16384, kvd.OPT_MAX_CTAS: 0}),
                       ("ce", {kvd.OPT_VARIANT: kvd.VARIANT_CE})):
        for k, v in opts.items():
            peer.set(k, v)
        table[:] = [c_s, c_d] if name == "ce" else [s_ids, d_ids]
        # drain completion slots between phases
        pulls(2)
        torch.cuda.synchronize(1)
        for r in range(1, rid[0] + 1):
            try:
                peer.poll(r)
            except kvd.KvdError:
                pass
        _, tp = timed(None, lambda: pulls(KP))
        alone = KP * bytes_per / tp / 1e9
        for r in range(1, rid[0] + 1):
            try:
                peer.poll(r)
            except kvd.KvdError:
                pass
        tg2, tp2 = timed(lambda: gemms(KG), lambda: pulls(KP))
        for r in range(1, rid[0] + 1):
            try:
                peer.poll(r)
            except kvd.KvdError:
                pass
        out[name] = {"pull_alone_gbs": round(alone, 1), "pull_with_gemm_gbs": round(KP * bytes_per / tp2 / 1e9, 1),
                     "gemm_with_pull_tflops": round(KG * flop / tg2 / 1e12, 1),
                     "gemm_slowdown": round(base_tflops / (KG * flop / tg2 / 1e12), 3)}
        print(json.dumps({name: out[name]}), flush=True)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
