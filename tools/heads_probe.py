#!/usr/bin/env python
"""§8 f4 bandwidth: decode shard of a TP=4 group (2 KV heads) pulls the two
prefill TP=8 shards (1 head each) into its head slices, C4 geometry (80
layers, head_dim 128, bf16, 8K tokens); vs the plain TP=4 -> TP=4 pull of the
same bytes.  GPU0 holds the prefill shards, GPU1 the decode cache."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import kvdgen
from paper_2501_14743_b200.torch_cache import PagedCache

NL, D, BS, NB, n = 80, 128, 16, 1024, 512
mk = lambda h, dev: PagedCache(NL, h, D, BS, NB, kvdgen.BF16, (0,) * 5, dev)
shards = [mk(1, 0), mk(1, 0)]
whole = mk(2, 0)
dst = mk(2, 1)
torch.cuda.synchronize(0)
s_ids, d_ids = kvdgen.fragmented_table(n, NB, NB, seed=4)
peers = [dst.open_peer_heads(c.export(), i) for i, c in enumerate(shards)]
# optional overrides, e.g. HEADS_OPTS="variant=4,threads=256,stages=6,ctas=148"
from paper_2501_14743_b200 import kvd
_OPT = {"variant": kvd.OPT_VARIANT, "threads": kvd.OPT_THREADS, "stages": kvd.OPT_STAGES,
        "ctas": kvd.OPT_MAX_CTAS, "tile": kvd.OPT_TILE_BYTES}
for kv in filter(None, os.environ.get("HEADS_OPTS", "").split(",")):
    k, v = kv.split("=")
    for p in peers:
        p.set(_OPT[k], int(v))
plain = dst.open_peer(whole.export())
st = torch.cuda.Stream(1)
rid = [0]


def run(ps, reps=20):
    def once():
        ids = []
        for p in ps:
            rid[0] += 1
            p.pull(rid[0], s_ids, d_ids, st)
            ids.append((p, rid[0]))
        for p, r in ids:
            p.wait(r)
    once()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        once()
    e1.record(st)
    torch.cuda.synchronize(1)
    return e0.elapsed_time(e1) / 1e3 / reps


nbytes = n * NL * 2 * BS * 2 * D * 2
t_h = run(peers)
t_p = run([plain])
print(json.dumps({"opts": os.environ.get("HEADS_OPTS", ""), "bytes": nbytes, "tp8_to_tp4_head_slices_gbs": round(nbytes / t_h / 1e9, 1),
                  "launches": 2, "info": peers[0].info(),
                  "tp4_to_tp4_plain_gbs": round(nbytes / t_p / 1e9, 1)}))
