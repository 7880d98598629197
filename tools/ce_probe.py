#!/usr/bin/env python
"""Copy-engine vs SM pull ceiling over NVLink for large contiguous transfers:
torch peer copies issued from the destination's or the source's stream, and
the kvd pull (TMA ring / LSU) over the same sizes."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import kvdgen
from paper_2501_14743_b200 import kvd
from paper_2501_14743_b200.torch_cache import PagedCache


def timeit(fn, stream, reps=3):
    fn(); torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    return e0.elapsed_time(e1) / 1e3 / reps


for gib in (1, 4, 16, 32):
    n = gib << 30
    x = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    y = torch.empty(n, dtype=torch.uint8, device="cuda:1")
    s_dst, s_src = torch.cuda.Stream(1), torch.cuda.Stream(0)
    def on_dst():
        with torch.cuda.stream(s_dst):
            y.copy_(x, non_blocking=True)
    def on_src():
        with torch.cuda.stream(s_src):
            y.copy_(x, non_blocking=True)
    t1 = timeit(on_dst, s_dst); t2 = timeit(on_src, s_src)
    print(json.dumps({"gib": gib, "ce_issued_on_dst_gbs": round(n / t1 / 1e9, 1),
                      "ce_issued_on_src_gbs": round(n / t2 / 1e9, 1)}), flush=True)
    del x, y
    torch.cuda.empty_cache()

g = kvdgen.C2.with_blocks(4096)   # 32 GiB per side
src = PagedCache(g.num_layers, g.num_kv_heads, g.head_dim, g.block_size, g.num_blocks, g.dtype, g.stride, 0)
dst = PagedCache(g.num_layers, g.num_kv_heads, g.head_dim, g.block_size, g.num_blocks, g.dtype, g.stride, 1)
torch.cuda.synchronize(0)
peer = dst.open_peer(src.export())
st = torch.cuda.Stream(1)
rid = [0]
for nb in (512, 2048, 4096):
    s, d = kvdgen.contiguous_table(nb)
    for name, var in (("auto", 0), ("lsu32", 2), ("ce", 3)):
        peer.set(kvd.OPT_VARIANT, var)
        def go():
            rid[0] += 1
            peer.pull(rid[0], s, d, st)
            peer.wait(rid[0])
        t = timeit(go, st)
        print(json.dumps({"blocks": nb, "bytes": nb * 8 << 20, "mover": name, "ctas": peer.info()["ctas"],
                          "gbs": round(nb * (8 << 20) / t / 1e9, 1)}), flush=True)
