#!/usr/bin/env python
"""Timeline of back-to-back single pulls from the in-kernel %globaltimer
(KVD_OPT_TIMING = 2: no events between launches, so programmatic dependent
launch overlaps consecutive pulls as in the bench).  Per request:

  span    = last CTA done - first CTA start          (the kernel's own time)
  pre     = return from griddepcontrol.wait - start (early source reads
            overlapping the previous pull; 0 without early loads)
  period  = end(k) - end(k-1)                        (steady-state cost per request)
  handoff = wait(k) - end(k-1)                       (previous pull's completion
            -> this pull may store: grid drain, memory flush, PDL release)

    python tools/timeline.py --config c4 --tokens 128,1024 --requests 32 [--early 0]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--src-dev", type=int, default=0)
    ap.add_argument("--dst-dev", type=int, default=1)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--tokens", default="128,1024")
    ap.add_argument("--requests", type=int, default=32)
    ap.add_argument("--early", type=int, default=1)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--label", default="")
    a = ap.parse_args()
    base = {"c1": kvdgen.C1, "c2": kvdgen.C2, "c4": kvdgen.C4}[a.config]
    toks = [int(t) for t in a.tokens.split(",")]
    need = max(kvdgen.blocks_for(t, base.block_size) for t in toks) * a.requests
    g = base.with_blocks(max(need * 6 // 5 + 64, 256))
    mk = lambda dev: PagedCache(g.num_layers, g.num_kv_heads, g.head_dim, g.block_size,
                                g.num_blocks, g.dtype, g.stride, dev)
    src, dst = mk(a.src_dev), mk(a.dst_dev)
    for l in range(g.num_layers):
        kvdgen.torch_fill_random_(src.layers[l], 10 + l)
    torch.cuda.synchronize(a.src_dev)
    peer = dst.open_peer(src.export())
    peer.set(kvd.OPT_EARLY_LOADS, a.early).set(kvd.OPT_TIMING, 2)
    for opt, v in ((kvd.OPT_MAX_CTAS, a.ctas), (kvd.OPT_STAGES, a.stages),
                   (kvd.OPT_TILE_BYTES, a.tile), (kvd.OPT_THREADS, a.threads),
                   (kvd.OPT_VARIANT, a.variant)):
        if v:
            peer.set(opt, v)
    torch.cuda.set_device(a.dst_dev)
    stream = torch.cuda.Stream(a.dst_dev)
    rid = 0
    for t in toks:
        n = kvdgen.blocks_for(t, g.block_size)
        tables = kvdgen.disjoint_fragmented_tables([n] * a.requests, g.num_blocks, g.num_blocks,
                                                   seed=t)
        per = n * g.num_layers * 2 * src.span_bytes
        rows = []
        for it in range(3):
            with torch.cuda.stream(stream):
                torch.cuda._sleep(2_000_000)            # host issue hidden behind ~1 ms
            ids = []
            for s, d in tables:
                rid += 1
                peer.pull(rid, s, d, stream)
                ids.append(rid)
            for r in ids:
                peer.wait(r)
            sp = sorted(peer.spans(), key=lambda x: x[3])
            if it:
                rows.append(sp)
        st = {"span": [], "pre": [], "period": [], "handoff": []}
        for sp in rows:
            for k, (r, s0, w, e) in enumerate(sp):
                st["span"].append(e - s0)
                st["pre"].append(w - s0)
                if k:
                    st["period"].append(e - sp[k - 1][3])
                    st["handoff"].append(w - sp[k - 1][3])
        med = {k: round(float(np.median(v)) / 1e3, 2) for k, v in st.items()}
        res = {"label": a.label, "config": a.config, "tokens": t, "bytes_per_request": per,
               "early": a.early, "info": {k: peer.info()[k] for k in ("variant", "ctas", "threads",
                                                                     "runs", "tiles")},
               "us_median": med,
               "gbs_per_period": round(per / (med["period"] * 1e3), 1),
               "gbs_per_span": round(per / (med["span"] * 1e3), 1),
               "opts": {"ctas": a.ctas, "stages": a.stages, "tile": a.tile,
                        "threads": a.threads}}
        print(json.dumps(res), flush=True)
    peer.close()
    dst.close()
    src.close()


if __name__ == "__main__":
    main()
