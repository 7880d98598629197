#!/usr/bin/env python
"""bench.py -- KV pull GB/s per GPU pair and p50 per-request transfer latency
(BASELINE.json metric) for KVDirect's pull path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1|c3|c4]
                    [--table fragmented|contiguous|worst] [--batch] [--impl kvd|reference]

N = 1: no NVLink pair exists on one GPU, so the prefill and decode caches
share cuda:0 (loopback pull, HBM-bound); this is stated in config.pairing.
N >= 2 (torchrun, one process per GPU): ranks [0, N/2) hold prefill caches,
ranks [N/2, N) decode caches; decode rank N/2 + k pulls from prefill rank k
(the paper's rail rule "GPU i ... only with GPU i") over NVLink 5
/ NVSwitch through CUDA IPC.  No collective on the data path.

A step = one pass of the per-request hot path over
one batch of synthetic input on every pair: kvd_pull per request (validate +
coalesce + one launch) -- or one kvd_pull_batch for the whole batch with
--batch (§8 f1) -- and kvd_poll_done until every request's device-side
completion word flips.  C1/C2/C4: one request per pair per step; C3: the
pair's 16 mixed-length requests.  Rows a1-a2 (register, export/open) are the
paper's one-time Connect() and run before the timed region.  The K steps
are issued back to back (a serving engine posts each pull as its request
arrives) and completions retired as they land.
`value` = bytes pulled by all pairs / device time of the K steps (CUDA events
on the pull stream, max over ranks); `e2e` = the same bytes / host wall time
from the first kvd_pull entry to the last completion observed;
`roofline.achieved` = algorithmic bytes per launch / average launch duration,
the latter from the CUDA events over the timed region on the pull stream
(which holds nothing but back-to-back pull launches), cross-checked by the
in-kernel %globaltimer span of every launch (KVD_OPT_TIMING = 2: no events
between launches); `--timing events` instead brackets every launch with
library events (KVD_OPT_TIMING = 1); `p50_latency_ms` = issue -> completion
observed of single requests on an idle pair, measured after the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import kvdgen  # noqa: E402

METRIC = "KV pull GB/s per GPU pair vs 900 GB/s NVLink; p50 per-request transfer latency"
NVLINK_NOMINAL_GBS = 900.0
NVLINK_MEASURED_GBS = 770.0   # B200_PROFILING.md: measured peer copy per direction
# NVLink 5 read user-data ceiling: 900 GB/s per direction on the wire, of which
# every 128 B read response carries 16 B of protocol (ncu nvlrx__bytes_data_protocol
# = 1/8 of nvlrx__bytes_data_user, profiles/ncu_pull_c2_nvlink.json) -> 900 * 128 / 144
NVLINK_READ_USER_GBS = NVLINK_NOMINAL_GBS * 128.0 / 144.0
C3_PAIRS = 4                  # C3 is defined on 4P:4D pairs; pair k gets requests i % 4 == k


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------

def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback B200_PROFILING.md"


def nearest_rank(xs, q):
    """Nearest-rank percentile."""
    s = sorted(xs)
    if not s:
        return None
    k = max(1, int(np.ceil(q / 100.0 * len(s))))
    return s[k - 1]


class ClockSampler:
    """Samples SM clock and clock-event reasons through NVML during the
    timed region (B200_PROFILING.md clocks line)."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[device_index]) if vis else device_index
            self._h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self._nvml = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            # first queries outside the timed region (the first call of each
            # is the slow one)
            pynvml.nvmlDeviceGetClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            self._nvml = None
        self.period = period_s

    def _run(self):
        n = self._nvml
        while not self._stop.is_set():
            try:
                self.samples.append(n.nvmlDeviceGetClockInfo(self._h, n.NVML_CLOCK_SM))
                r = n.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._nvml:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
                "reasons": sorted(self.reasons)}


DESC = {
    "c1": "C1 tiny (2 layers, 2 KV heads, head_dim 64, block 16, fp16), one 256-token request",
    "c2": "C2 Llama-2-7B KV cache (32 layers, 32 KV heads, head_dim 128, block 16, fp16), "
          "one 8K-token request",
    "c3": "C3 Llama-2-7B, 64 mixed-length requests U{512..8192} tokens (random.Random(0)), "
          "fragmented block tables, 16 requests per pair (request i -> pair i % 4)",
    "c4": "C4 Llama-3-70B TP=4 shard (80 layers, 2 KV heads/shard, head_dim 128, block 16, "
          "bf16), one 8K-token request per shard",
}


def workload(config: str, table: str, pair_index: int = 0):
    """(geometry, [(src_ids, dst_ids)] for this pair, description)."""
    if config == "c3":
        toks = kvdgen.mixed_request_tokens(kvdgen.C3_REQUESTS, seed=0)
        mine = [t for i, t in enumerate(toks) if i % C3_PAIRS == pair_index % C3_PAIRS]
        counts = [kvdgen.blocks_for(t, 16) for t in mine]
        pool = 6144
        g = kvdgen.C2.with_blocks(pool)
        reqs = kvdgen.disjoint_fragmented_tables(counts, pool, pool, seed=3 + pair_index)
        return g, reqs, DESC["c3"]
    if config == "c1":
        g, tokens = kvdgen.C1, kvdgen.C1_TOKENS
    elif config == "c4":
        g, tokens = kvdgen.C4, kvdgen.C4_TOKENS
    else:
        g, tokens = kvdgen.C2, kvdgen.C2_TOKENS
    n = kvdgen.blocks_for(tokens, g.block_size)
    if table == "contiguous":
        s, d = kvdgen.contiguous_table(n, 0, g.num_blocks - n)
    elif table == "worst":
        s, d = kvdgen.fixed_run_table(n, 1, g.num_blocks, g.num_blocks, seed=1)
    else:
        s, d = kvdgen.fragmented_table(n, g.num_blocks, g.num_blocks, seed=1)
    return g, [(s, d)], DESC.get(config, DESC["c2"])


def cpu_oracle_sample(target_s: float = 12.0):
    """Time the CPU oracle (oracle/kvd_oracle.c, single thread, as it stands)
    on a bounded sample of the C2 workload: C2 geometry, a fragmented request
    of k blocks drawn from pools of 2k blocks, k chosen to take ~target_s."""
    from oracle import oracle
    g = kvdgen.C2

    def run(k):
        nb = 2 * k
        lb = oracle.layer_nbytes((0,) * 5, nb, g.block_size, g.num_kv_heads, g.head_dim, 2)
        src = [kvdgen.random_bytes(lb, 10 + l) for l in range(g.num_layers)]
        dst = [np.zeros(lb, np.uint8) for _ in range(g.num_layers)]
        s, d = kvdgen.fragmented_table(k, nb, nb, seed=2)
        t = time.perf_counter()
        rc = oracle.pull(src, (0,) * 5, nb, dst, (0,) * 5, nb, g.num_kv_heads, g.head_dim,
                         g.block_size, 2, s, d)
        dt = time.perf_counter() - t
        assert rc == 0
        return dt, k * g.num_layers * 2 * g.block_size * g.num_kv_heads * g.head_dim * 2

    def run_all_cores(k, threads):
        """The same oracle call, one host thread per group of layers (ctypes
        releases the GIL inside the C loop): the oracle as it stands, on every
        core of the box."""
        from concurrent.futures import ThreadPoolExecutor
        nb = 2 * k
        lb = oracle.layer_nbytes((0,) * 5, nb, g.block_size, g.num_kv_heads, g.head_dim, 2)
        src = [kvdgen.random_bytes(lb, 10 + l) for l in range(g.num_layers)]
        dst = [np.zeros(lb, np.uint8) for _ in range(g.num_layers)]
        s, d = kvdgen.fragmented_table(k, nb, nb, seed=2)
        groups = [list(range(i, g.num_layers, threads)) for i in range(threads)]
        groups = [x for x in groups if x]

        def part(ls):
            return oracle.pull([src[l] for l in ls], (0,) * 5, nb, [dst[l] for l in ls], (0,) * 5,
                               nb, g.num_kv_heads, g.head_dim, g.block_size, 2, s, d)
        t = time.perf_counter()
        with ThreadPoolExecutor(len(groups)) as ex:
            assert all(rc == 0 for rc in ex.map(part, groups))
        dt = time.perf_counter() - t
        return dt, k * g.num_layers * 2 * g.block_size * g.num_kv_heads * g.head_dim * 2, len(groups)

    dt, b = run(2)
    k = int(max(2, min(256, 2 * target_s / max(dt, 1e-3))))
    dt, b = run(k)
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    adt, ab, used = run_all_cores(k, min(ncpu, g.num_layers))
    return {"value": round(b / dt / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
            "seconds": round(dt, 2),
            "sample": f"C2 geometry, fragmented {k}-block request ({b / 2**20:.0f} MiB) from "
                      f"{2 * k}-block pools, oracle/kvd_oracle.c element loop, 1 thread",
            "all_cores": {"value": round(ab / adt / 1e9, 4), "unit": "GB/s", "cores": used,
                          "seconds": round(adt, 2),
                          "what": "same sample, layers split over host threads"}}


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle (tier rule: the oracle is the reference)
# ---------------------------------------------------------------------------

def run_reference(args, rank, world):
    if rank != 0:
        return
    from oracle import oracle
    g, reqs, desc = workload(args.config, args.table)
    k = 4 if args.config != "c1" else len(reqs[0][0])
    nb = max(2 * k, 8)
    g = g.with_blocks(nb)
    lb = oracle.layer_nbytes((0,) * 5, nb, g.block_size, g.num_kv_heads, g.head_dim,
                             g.elem_bytes)
    src = [kvdgen.random_bytes(lb, 10 + l) for l in range(g.num_layers)]
    dst = [np.zeros(lb, np.uint8) for _ in range(g.num_layers)]
    s, d = kvdgen.fragmented_table(k, nb, nb, seed=2)
    per = k * g.num_layers * 2 * g.block_size * g.num_kv_heads * g.head_dim * g.elem_bytes

    def step():
        rc = oracle.pull(src, (0,) * 5, nb, dst, (0,) * 5, nb, g.num_kv_heads, g.head_dim,
                         g.block_size, g.elem_bytes, s, d)
        assert rc == 0

    for _ in range(args.warmup):
        step()
    lat = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        t = time.perf_counter()
        step()
        lat.append(time.perf_counter() - t)
    dt = time.perf_counter() - t0
    value = per * args.steps / dt / 1e9
    sample = (f"{desc}: bounded sample of {k} blocks ({per / 2**20:.1f} MiB) per step from "
              f"{nb}-block host pools, oracle/kvd_oracle.c element loop, 1 thread")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": desc, "sample_blocks": k},
        "p50_latency_ms": round(nearest_rank(lat, 50) * 1e3, 3),
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": 1,
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
# the pull arm
# ---------------------------------------------------------------------------

def nvlink_rx_from_profile(config: str):
    """NVLink receive counters of the decode GPU from the committed ncu
    summary (profiles/ncu_pull_<config>_nvlink.json): user data vs total
    bytes per launch and their rates over the profiled kernel's duration."""
    p = os.path.join(ROOT, "profiles", f"ncu_pull_{config}_nvlink.json")
    try:
        with open(p) as f:
            m = json.load(f)["metrics"]
        t = m["gpu__time_duration.sum"]["value"] * 1e-6
        user = m["nvlrx__bytes_data_user.sum"]["value"]
        total = m["nvlrx__bytes.sum"]["value"]
        return {"user_bytes": int(user), "total_bytes": int(total),
                "user_gbs": round(user / t / 1e9, 1), "total_gbs": round(total / t / 1e9, 1),
                "protocol_frac": round(1 - user / total, 4),
                "source": os.path.relpath(p, ROOT) + " (ncu --set full, one launch, cold)"}
    except Exception:
        return None


def traffic_from_profile(config: str, nvlink: bool):
    """dram bytes per launch of the pull kernel from the committed ncu
    --set full summary (profiles/ncu_pull_<config>[_nvlink].json), else None.
    For the NVLink case this is the decode GPU's DRAM only (the prefill
    GPU's reads are not visible to the decode process's counters)."""
    p = os.path.join(ROOT, "profiles", f"ncu_pull_{config}{'_nvlink' if nvlink else ''}.json")
    try:
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


def decode_matches(dst, g, s_ids, d_ids, src_seed, dst_seed, dev, scribble_seed=None):
    """Element-wise parity of a whole decode cache: layer l must equal its
    seeded pre-state (seed dst_seed*1000+l, or scribble_seed+l after a
    baseline scribbled it) with blocks d_ids replaced by the prefill's blocks
    s_ids (seed src_seed*1000+l), for every layer, K/V plane and byte."""
    import torch
    span = dst.span_bytes
    si = torch.from_numpy(np.ascontiguousarray(s_ids)).long().cuda(dev)
    di = torch.from_numpy(np.ascontiguousarray(d_ids)).long().cuda(dev)
    ok = True
    for l in range(g.num_layers):
        exp = torch.empty_like(dst.layers[l])
        kvdgen.torch_fill_random_(exp, (scribble_seed + l) if scribble_seed is not None
                                  else dst_seed * 1000 + l)
        srcl = torch.empty_like(dst.layers[l])
        kvdgen.torch_fill_random_(srcl, src_seed * 1000 + l)
        exp.view(2, g.num_blocks, span)[:, di] = srcl.view(2, g.num_blocks, span)[:, si]
        ok = ok and bool(torch.equal(dst.layers[l], exp))
        del exp, srcl
    torch.cuda.synchronize(dev)
    return ok


def nccl_baselines(args, g, reqs, src, dst, role, rank, half, dev, gloo, src_seed):
    """The measured baseline (north_star: "NCCL send/recv is kept only as the
    measured baseline"), same caches and block tables as the pull.

    N1 = the message-passing flow of fig:diff(a): decode sends the
    wanted block ids (step 1), prefill gathers the blocks into a staging
    buffer with a kernel (2) and ncclSend's it (3), decode ncclRecv's and
    scatters it into its paged cache (4).  The whole step is staged at once
    (one message per step: favourable to NCCL).
    N2 = grouped per-segment send/recv (ncclGroupStart/End via
    batch_isend_irecv), no staging: one send/recv per contiguous (layer,
    K/V, run) segment straight between the paged caches (C1/C2/C4 only).
    N3 = N1 with a BOUNDED communication buffer, the way fig:diff(a) drives
    it: the block list is cut into chunks, two staging buffers
    alternate, and chunk k+1 is gathered (prefill) / chunk k-1 scattered
    (decode) while chunk k is on the wire; swept over chunk sizes.
    N0 = one contiguous ncclSend/ncclRecv of the same byte count: NCCL's
    own link ceiling, no paged layout at all (context, not a transfer of
    the cache).
    Each is timed as host wall per step (max over ranks) and parity-checked
    element by element (the decode cache is scribbled before each
    baseline; N0's received buffer is compared with its regenerated
    contents)."""
    import torch
    import torch.distributed as dist
    from paper_2501_14743_b200 import kvd
    s_ids = np.ascontiguousarray(np.concatenate([s for s, _ in reqs]), dtype=np.int32)
    d_ids = np.ascontiguousarray(np.concatenate([d for _, d in reqs]), dtype=np.int32)
    n = len(s_ids)
    span = (src or dst).span_bytes
    nb = g.num_blocks
    per = g.num_layers * 2 * n * span
    peer_rank = rank + half if role == "prefill" else rank - half
    stream = torch.cuda.current_stream(dev)
    ids_dev = torch.empty(n, dtype=torch.int32, device=f"cuda:{dev}")
    ids_host = torch.from_numpy(s_ids).pin_memory()
    out = {}

    def scribble():
        if role == "decode":
            for l, t in enumerate(dst.layers):
                kvdgen.torch_fill_random_(t, 777 + l)
        torch.cuda.synchronize(dev)

    staging = torch.empty(per, dtype=torch.uint8, device=f"cuda:{dev}")

    def n1():
        if role == "decode":
            ids_dev.copy_(ids_host, non_blocking=True)
            dist.send(ids_dev, peer_rank)
            dist.recv(staging, peer_rank)
            kvd.kvd_scatter(dst.handle, d_ids, staging.data_ptr(), stream.cuda_stream)
        else:
            dist.recv(ids_dev, peer_rank)
            want = ids_dev.cpu().numpy()          # the RPC'd block ids drive the gather
            kvd.kvd_gather(src.handle, want, staging.data_ptr(), stream.cuda_stream)
            dist.send(staging, peer_rank)
        torch.cuda.synchronize(dev)

    plans = [("n1_gather_send_recv_scatter", n1, args.steps)]
    seg_views = []
    if len(reqs) == 1 and not getattr(args, "no_n2", False):
        runs = kvd.kvd_plan(s_ids, d_ids, nb, nb)
        cache, side = (src, 0) if role == "prefill" else (dst, 1)
        for l in range(g.num_layers):
            layer = cache.layers[l]
            for p in range(2):
                for r in runs:
                    off = p * nb * span + int(r[side]) * span
                    seg_views.append(layer[off:off + int(r[2]) * span])

        def n2():
            if role == "decode":
                ids_dev.copy_(ids_host, non_blocking=True)
                dist.send(ids_dev, peer_rank)
                ops = [dist.P2POp(dist.irecv, v, peer_rank) for v in seg_views]
            else:
                dist.recv(ids_dev, peer_rank)
                ops = [dist.P2POp(dist.isend, v, peer_rank) for v in seg_views]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            torch.cuda.synchronize(dev)

        plans.append(("n2_grouped_segment_send_recv", n2, max(3, min(args.steps, 10))))

    unit = g.num_layers * 2 * span                 # bytes of one block, all layers and K/V

    def n3(cb):
        bounds = [(a, min(a + cb, n)) for a in range(0, n, cb)]
        bufs = [staging[:cb * unit], staging[cb * unit:2 * cb * unit]]

        def fn():
            works = []
            if role == "decode":
                ids_dev.copy_(ids_host, non_blocking=True)
                dist.send(ids_dev, peer_rank)
                for k, (a, b) in enumerate(bounds):
                    # the NCCL stream waits for the current stream here, i.e.
                    # for the scatter of chunk k-2 that read this buffer
                    works.append(dist.irecv(bufs[k % 2][:(b - a) * unit], peer_rank))
                    if k >= 1:
                        works[k - 1].wait()        # current stream after recv k-1
                        pa, pb = bounds[k - 1]
                        kvd.kvd_scatter(dst.handle, d_ids[pa:pb], bufs[(k - 1) % 2].data_ptr(),
                                        stream.cuda_stream)
                works[-1].wait()
                pa, pb = bounds[-1]
                kvd.kvd_scatter(dst.handle, d_ids[pa:pb], bufs[(len(bounds) - 1) % 2].data_ptr(),
                                stream.cuda_stream)
            else:
                dist.recv(ids_dev, peer_rank)
                want = ids_dev.cpu().numpy()
                for k, (a, b) in enumerate(bounds):
                    if k >= 2:
                        works[k - 2].wait()        # send k-2 has read this buffer
                    kvd.kvd_gather(src.handle, want[a:b], bufs[k % 2].data_ptr(),
                                   stream.cuda_stream)
                    works.append(dist.isend(bufs[k % 2][:(b - a) * unit], peer_rank))
                for w in works:
                    w.wait()
            torch.cuda.synchronize(dev)
        return fn

    chunk_sizes = sorted({max(1, (mib << 20) // unit) for mib in (64, 256, 1024)})
    for cb in chunk_sizes:
        if 2 * cb <= n:
            plans.append((f"n3_pipelined_{cb}_blocks", n3(cb), max(3, min(args.steps, 10))))

    def n0():
        if role == "decode":
            dist.recv(staging, peer_rank)
        else:
            dist.send(staging, peer_rank)
        torch.cuda.synchronize(dev)

    plans.append(("n0_raw_contiguous", n0, max(3, min(args.steps, 10))))

    for name, fn, steps in plans:
        scribble()
        if name.startswith("n0") and role == "prefill":
            kvdgen.torch_fill_random_(staging, 4242)
            torch.cuda.synchronize(dev)
        for _ in range(2):
            fn()
        dist.barrier()
        lat = []
        t0 = time.perf_counter()
        for _ in range(steps):
            t = time.perf_counter()
            fn()
            lat.append(time.perf_counter() - t)
        wall = time.perf_counter() - t0
        dist.barrier()
        ok = True
        if role == "decode":
            if name.startswith("n0"):
                exp = torch.empty_like(staging)
                kvdgen.torch_fill_random_(exp, 4242)
                ok = bool(torch.equal(exp, staging))
                del exp
            else:
                ok = decode_matches(dst, g, s_ids, d_ids, src_seed, None, dev, scribble_seed=777)
        out[name] = {"wall_s": wall, "steps": steps, "bytes": per * steps if role == "decode" else 0,
                     "lat": lat, "ok": ok,
                     "segments": (len(seg_views) if name.startswith("n2") else
                                  -(-n // int(name.split("_")[2])) if name.startswith("n3") else 1)}
    del staging
    return out


def run_kvd(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2501_14743_b200 import cluster, kvd
    from paper_2501_14743_b200.torch_cache import PagedCache

    torch.cuda.set_device(local_rank)
    dev = local_rank
    multi = world > 1
    ring = args.pairing == "ring" and multi
    if ring and not args.no_nccl:
        args.no_nccl = True            # the NCCL comparators assume prefill/decode halves
    me = cluster.ring_role_of(rank, world) if ring else cluster.role_of(rank, world)
    role, pairs, half = me.role, me.pairs, world // 2
    pair_index = (rank if ring else rank % half) if multi else 0
    g, reqs, desc = workload(args.config, args.table, pair_index)
    n_req = len(reqs)
    n_blocks = sum(len(s) for s, _ in reqs)
    gloo = dist.new_group(backend="gloo") if multi else None

    def new_cache(seed):
        c = PagedCache(g.num_layers, g.num_kv_heads, g.head_dim, g.block_size, g.num_blocks,
                       g.dtype, g.stride, dev, memory=args.memory)
        for l, t in enumerate(c.layers):
            kvdgen.torch_fill_random_(t, seed * 1000 + l)
        return c

    src = new_cache(1 + rank) if role in ("prefill", "both") else None
    dst = new_cache(100 + rank) if role in ("decode", "both") else None
    torch.cuda.synchronize()

    # row a2: one-time tensor-centric exchange (Connect())
    if multi:
        blob = cluster.peer_blob(me, cluster.exchange_blobs(src.export() if src else None, gloo))
    else:
        blob = src.export()
    peer = dst.open_peer(blob) if dst else None
    if peer:
        if args.variant:
            peer.set(kvd.OPT_VARIANT, {"lsu": 1, "lsu32": 2, "ce": 3, "tma": 4}[args.variant])
        if args.stages:
            peer.set(kvd.OPT_STAGES, args.stages)
        if args.tile:
            peer.set(kvd.OPT_TILE_BYTES, args.tile)
        if args.threads:
            peer.set(kvd.OPT_THREADS, args.threads)
        if args.max_ctas:
            peer.set(kvd.OPT_MAX_CTAS, args.max_ctas)
        if args.no_coalesce:
            peer.set(kvd.OPT_COALESCE, 0)
        if args.streams:
            peer.set(kvd.OPT_STREAMS, args.streams)
        if args.early is not None:
            peer.set(kvd.OPT_EARLY_LOADS, args.early)

    stream = torch.cuda.Stream(dev)
    rid = [rank * 10_000_000]
    launches = [0]

    pending = {}          # request id -> host issue time (ns)

    def issue(evs=None):
        """Rows a3-a4 for this pair's requests of one step: validate,
        coalesce and launch (kvd_pull per request, or one kvd_pull_batch);
        returns immediately ("post ... without block").  `evs`
        brackets the step's launches on the pull stream."""
        if evs is not None:
            evs[0].record(stream)
        if args.batch:
            ids = [rid[0] + 1 + q for q in range(n_req)]
            rid[0] += n_req
            t0 = time.perf_counter_ns()
            peer.pull_batch(ids, reqs, stream)
            for i in ids:
                pending[i] = t0
            launches[0] += 1
        else:
            for s, d in reqs:
                rid[0] += 1
                pending[rid[0]] = time.perf_counter_ns()
                peer.pull(rid[0], s, d, stream)
                launches[0] += 1
        if evs is not None:
            evs[1].record(stream)

    def retire(until, lat_out=None):
        """Row a6: poll completion words until at most `until` requests are
        in flight."""
        while len(pending) > until:
            for i in peer.poll_many(list(pending)):   # one C call for every pending request
                t0 = pending.pop(i)
                if lat_out is not None:
                    lat_out.append(time.perf_counter_ns() - t0)

    def step(lat_out=None):
        if lat_out is not None and n_req == 1 and not args.batch:
            # one request: issue -> completion observed by kvd_wait_done's C-side
            # spin on the slot word (no Python polling granularity in the number)
            s, d = reqs[0]
            rid[0] += 1
            t0 = time.perf_counter_ns()
            peer.pull(rid[0], s, d, stream)
            peer.wait(rid[0])
            lat_out.append(time.perf_counter_ns() - t0)
            return
        issue()
        retire(0, lat_out)

    def barrier():
        # a host-side (gloo) barrier: an NCCL barrier would leave a spinning
        # NCCL kernel on the prefill GPU for the whole timed region
        torch.cuda.synchronize()
        if multi:
            dist.barrier(group=gloo)

    # Everything the timed region needs is set up BEFORE the warm-up (NVML
    # init can take tens of ms): the GPU goes from the warm-up steps through
    # the barrier into the timed steps without an idle gap in which its
    # clocks or links could settle (a gap made the first timed C4 pulls
    # ~70 us slower in total, profiles/r02_c4_steps.txt).
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(K)] if peer and args.timing == "events" else []
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    lat_ns = []
    sampler = ClockSampler(dev)
    if peer:
        # timer: in-kernel %globaltimer spans only (events between launches would
        # block programmatic dependent launch); events: library events around each launch
        peer.set(kvd.OPT_TIMING, 1 if args.timing == "events" else 2)
    for _ in range(args.warmup):
        if peer:
            step()
    if peer:                           # the warm-up's spans and events are not the region's
        peer.device_time()
        if args.timing == "events":
            peer.kernel_time()
    launches[0] = 0
    barrier()
    # Throughput: the K steps are issued back to back, as a serving engine
    # posts each request's pull when it arrives; completions are retired as
    # they land (at most ~512 requests in flight, well under the 1024 slots).
    with sampler:
        wall0 = time.perf_counter()
        if peer:
            t_start.record(stream)
            for k in range(K):
                # timer mode: no events between launches (they would keep
                # programmatic dependent launch from overlapping consecutive pulls)
                issue(ev[k] if args.timing == "events" and not args.streams else None)
                if len(pending) > 768:
                    retire(512)
            if args.streams:
                peer.stream_wait(stream)   # join the library streams before the end event
            t_end.record(stream)
            retire(0)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    barrier()
    timed_launches = launches[0]
    kern_ms_total, kern_launches = (peer.kernel_time() if peer and args.timing == "events"
                                    else (0.0, 0))
    # %globaltimer cross-check (first CTA start -> last CTA done, single pulls
    # only; batches have no whole-launch arrival)
    gt_ms_total, gt_launches = peer.device_time() if peer else (0.0, 0)
    if peer:
        peer.set(kvd.OPT_TIMING, 0)
    # Per-request transfer latency (R16, SURVEY §8 d), after the timed region:
    # ISOLATED requests -- issue -> completion observed (kvd_wait_done's
    # C-side spin on the slot word) -> next, on an otherwise idle pair; all
    # pairs start each request together (gloo barrier), so for C4 the shards
    # of one request are pulled concurrently and its latency is the max over
    # the shard ranks.  C3 also reports the latency of requests queued as in
    # the timed steps (issue the pair's 16, retire as they land).
    if args.streams and peer:
        peer.set(kvd.OPT_STREAMS, 0)   # latency, parity and calibration in stream order
    reps = max(3, min(K, 50 if n_req == 1 else 3))
    for _ in range(reps):
        for s_, d_ in reqs:
            if multi:
                dist.barrier(group=gloo)
            if peer:
                rid[0] += 1
                t0 = time.perf_counter_ns()
                peer.pull(rid[0], s_, d_, stream)
                peer.wait(rid[0])
                lat_ns.append(time.perf_counter_ns() - t0)
    lat_queued = []
    if peer and n_req > 1:
        for _ in range(3):
            step(lat_queued)
    # --engine C: the same isolated requests posted to the resident pull
    # engine (KVD_OPT_ENGINE; no launch per request, not stream-ordered)
    lat_engine = []
    if args.engine:
        if peer:
            peer.set(kvd.OPT_ENGINE, args.engine)
        for _ in range(reps):
            for s_, d_ in reqs:
                if multi:
                    dist.barrier(group=gloo)
                if peer:
                    rid[0] += 1
                    t0 = time.perf_counter_ns()
                    peer.pull(rid[0], s_, d_, stream)
                    peer.wait(rid[0])
                    lat_engine.append(time.perf_counter_ns() - t0)
        if peer:
            peer.set(kvd.OPT_ENGINE, 0)

    info = peer.info() if peer else {}
    dev_s = t_start.elapsed_time(t_end) / 1e3 if peer else 0.0
    step_ms = ([a.elapsed_time(b) for a, b in ev] if args.timing == "events" and not args.streams
               else [dev_s * 1e3 / K] if peer else [])
    span = (src or dst).span_bytes
    bytes_per_step = n_blocks * g.num_layers * 2 * span

    # parity of the timed configuration (checked once, after timing),
    # element by element: every layer of the decode cache must equal the
    # plain definition of the result (SURVEY §8 c) -- its own seeded
    # pre-state with the requested blocks replaced by the prefill's blocks,
    # both regenerated here from their torch-generator seeds.
    s_all = np.concatenate([s for s, _ in reqs])
    d_all = np.concatenate([d for _, d in reqs])
    src_seed = 1 + (me.peer if multi else rank)
    ok = True
    if role in ("decode", "both"):
        ok = decode_matches(dst, g, s_all, d_all, src_seed, 100 + rank, dev)
    oks = [None] * world if multi else [ok]
    if multi:
        dist.all_gather_object(oks, bool(ok), group=gloo)

    # Link calibration (SURVEY §8 d; after the parity check, it overwrites
    # destination blocks): a CONTIGUOUS request as large as the first
    # request of a step, (i) read by the product's mover (auto policy: the
    # TMA ring over NVLink) -- what the fragmented block table costs -- and
    # (ii) copied by the copy engine over the same mapping (one
    # cudaMemcpyAsync per (layer, K/V) segment, KVD_VARIANT_CE).
    ce_gbs = tma_gbs = None
    if peer and args.config != "c1":
        n0 = min(len(reqs[0][0]), g.num_blocks)
        cs, cd = kvdgen.contiguous_table(n0, 0, g.num_blocks - n0)

        def timed_contiguous(reps=3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            rid[0] += 1
            peer.pull(rid[0], cs, cd, stream)
            peer.wait(rid[0])
            e0.record(stream)
            for _ in range(reps):
                rid[0] += 1
                peer.pull(rid[0], cs, cd, stream)
            e1.record(stream)
            peer.wait(rid[0])
            torch.cuda.synchronize()
            return reps * n0 * g.num_layers * 2 * span / (e0.elapsed_time(e1) / 1e3) / 1e9

        peer.set(kvd.OPT_VARIANT, kvd.VARIANT_CE)
        ce_gbs = timed_contiguous()
        peer.set(kvd.OPT_VARIANT, {"lsu": 1, "lsu32": 2, "ce": 3, "tma": 4}.get(args.variant, 0))
        tma_gbs = timed_contiguous()
    # The measured link ceiling (SURVEY §8 d, the calibration kernel): pure
    # bulk reads of the prefill cache through the same mapping, no stores
    # (kvd_peer_calibrate), best over grid sizes; the NVLink roofline's peak.
    read_ceiling = None
    if peer and multi and args.config != "c1":
        nbytes = min(g.num_layers * (dst.layer_bytes // 32768) * 32768, 2 << 30)
        read_ceiling = {f"{c}x{st}": peer.calibrate(nbytes, ctas=c, stages=st, reps=4)
                        for c in (48, 96, 148) for st in (6, 7)}

    base = {}
    if multi and not args.no_nccl:
        base = nccl_baselines(args, g, reqs, src, dst, role, rank, half, dev, gloo,
                              src_seed)

    stats = {"dev_s": dev_s, "wall_s": wall if peer else 0.0,
             "bytes": bytes_per_step * K if peer else 0,
             "step_ms": float(np.mean(step_ms)) if step_ms else 0.0,
             # per step: launch-bracketed library events, or the timed region's own
             # events divided by the steps (the region holds only pull launches)
             "kern_ms": ((kern_ms_total / K if args.timing == "events" else dev_s * 1e3 / K)
                         if peer else 0.0), "kern_launches": kern_launches,
             "gt_ms": gt_ms_total / gt_launches if gt_launches else 0.0,
             "gt_ms_total": gt_ms_total, "gt_launches": gt_launches,
             "lat": lat_ns, "clock": sampler.summary(), "info": info, "base": base,
             "launches": timed_launches, "runs": info.get("runs"), "ce_gbs": ce_gbs,
             "tma_gbs": tma_gbs, "read_ceiling": read_ceiling,
             "lat_queued": lat_queued, "lat_engine": lat_engine,
             "bytes_per_step": bytes_per_step if peer else 0}
    all_stats = cluster.gather_stats(stats, gloo) if multi else [stats]

    if rank == 0:
        dec = [s for s in all_stats if s["bytes"]]
        agg = cluster.aggregate(all_stats)          # max time / sum bytes over ranks
        t_dev, t_wall, total = agg["dev_s"], agg["wall_s"], agg["bytes"]
        lat_all = [x for s in dec for x in s["lat"]]
        # C4: one request = one block table pulled by every TP shard pair at
        # once; its latency is the slowest shard's (SURVEY §8 d)
        lat_req = ([max(col) for col in zip(*[s["lat"] for s in dec])]
                   if args.config == "c4" and len(dec) > 1 else lat_all)
        engine_req = ([max(col) for col in zip(*[s["lat_engine"] for s in dec])]
                      if args.config == "c4" and len(dec) > 1
                      else [x for s in dec for x in s["lat_engine"]])
        step_dev = max(s["step_ms"] for s in dec)
        info0 = dec[0]["info"]
        peaks, peak_src = measured_peaks()
        # roofline: each pair's bytes per step over its average step duration on
        # the pull stream (see the module docstring for the two timing modes)
        per_pair = [s["bytes_per_step"] / (s["kern_ms"] / 1e3) / 1e9 for s in dec]
        kern_dev = max(s["kern_ms"] for s in dec)
        achieved_link = float(np.mean(per_pair))
        bytes_per_step = dec[0]["bytes_per_step"]
        if multi:
            ceil = [max(s["read_ceiling"].values()) for s in dec if s["read_ceiling"]]
            measured = float(np.mean(ceil)) if len(ceil) == len(dec) else None
            peak = measured or NVLINK_READ_USER_GBS
            roof = {"bound": "nvlink", "achieved": round(achieved_link, 1),
                    "peak": round(peak, 1), "unit": "GB/s",
                    "frac": round(achieved_link / peak, 4),
                    "peak_source": ("measured in this run: kvd_peer_calibrate, discarded bulk "
                                    "(TMA) reads of the prefill cache through the same NVLink "
                                    "mapping, no stores, best of 48/96/148 CTAs x 6/7 stages of 32 KiB, "
                                    "mean over pairs"
                                    if measured else
                                    "NVLink 5 read user-data ceiling: 900 GB/s per direction x "
                                    "128/144 (16 B protocol per 128 B read response, measured by "
                                    "the ncu nvlrx counters in nvlink_rx)"),
                    "measured_read_ceiling": ({"per_pair": [{str(k): round(v, 1) for k, v in
                                                             s["read_ceiling"].items()}
                                                            for s in dec],
                                               "what": "GB/s by CTAs x ring stages"}
                                              if measured else None),
                    "frac_of_read_user_ceiling_800": round(achieved_link / NVLINK_READ_USER_GBS, 4),
                    "frac_of_guide_770": round(achieved_link / NVLINK_MEASURED_GBS, 4),
                    "frac_of_nominal_900": round(achieved_link / NVLINK_NOMINAL_GBS, 4),
                    "algorithmic_bytes_per_step": bytes_per_step,
                    "per_pair_achieved": [round(x, 1) for x in per_pair],
                    "traffic": traffic_from_profile(args.config, True),
                    "nvlink_rx": nvlink_rx_from_profile(args.config)}
            if all(s["gt_launches"] for s in dec):
                gt = [s["bytes"] / (s["gt_ms_total"] / 1e3) / 1e9 for s in dec]
                roof["globaltimer_cross_check"] = {
                    "achieved": round(float(np.mean(gt)), 1),
                    "ms_per_launch": round(float(np.mean([s["gt_ms"] for s in dec])), 4),
                    "what": "in-kernel %globaltimer, first CTA start -> last CTA done, "
                            "averaged over the timed launches (no launch latency)"}
        else:
            alg = 2 * bytes_per_step   # loopback: every byte is read and written in the same HBM
            roof = {"bound": "hbm", "achieved": round(alg / (kern_dev / 1e3) / 1e9, 1),
                    "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": round(alg / (kern_dev / 1e3) / 1e9 / peaks["hbm_gbs"], 4),
                    "peak_source": peak_src + " hbm_gbs (burst copy, read+write bytes)",
                    "algorithmic_bytes_per_step": alg,
                    "traffic": traffic_from_profile(args.config, False)}
            s0 = dec[0]
            if s0["gt_launches"]:
                roof["globaltimer_cross_check"] = {
                    "achieved": round(2 * s0["bytes"] / (s0["gt_ms_total"] / 1e3) / 1e9, 1),
                    "ms_per_launch": round(s0["gt_ms"], 4),
                    "what": "in-kernel %globaltimer, first CTA start -> last CTA done, "
                            "averaged over the timed launches (no launch latency)"}
        clk = all_stats[world // 2 if multi else 0]["clock"]
        out = {
            "metric": METRIC, "value": round(total / t_dev / 1e9, 2), "unit": "GB/s",
            "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": round(t_dev / K * 1e3, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {
                "workload": desc,
                "table": (f"{args.table} (kvdgen seed 1)" if args.config != "c3"
                          else "disjoint fragmented (kvdgen seed 3 + pair)"),
                "requests_per_pair_per_step": n_req, "blocks_per_pair_per_step": n_blocks,
                "bytes_per_pair_per_step": bytes_per_step, "runs": info0.get("runs"),
                "pairs": pairs,
                "pairing": ("loopback: prefill and decode caches on the same GPU (one GPU has "
                            "no NVLink pair)") if not multi else
                           (f"ring stress: every GPU holds both caches and rank k pulls from "
                            f"rank k+1 mod {world} over NVLink 5 ({pairs} concurrent pulls; "
                            f"every GPU's ingress and egress carry one)" if ring else
                            f"{pairs}P:{pairs}D rail pairs, rank k -> rank {pairs}+k over NVLink 5"),
                "parallelism": ("loopback" if not multi else
                                f"ring{pairs}" if ring else f"{pairs}x(1P:1D)"),
                "issue": ("kvd_pull_batch (one launch per step)" if args.batch
                          else "one kvd_pull per request")
                         + (f"; KVD_OPT_STREAMS={args.streams} (consecutive launches overlap "
                            "on library streams)" if args.streams else "; stream-ordered"),
                "l2": "no flush: every step moves >= 640 MiB per pair, >> 126 MB L2",
                "cache_dtype": "fp16" if g.dtype == kvdgen.FP16 else "bf16",
                "variant": info0.get("variant"), "ctas": info0.get("ctas"),
                "threads": info0.get("threads"), "tiles": info0.get("tiles"),
                "memory": ("torch caching allocator (cudaMalloc; legacy IPC handles)"
                           if args.memory == "torch" else
                           "kvd_mem_alloc (CUDA VMM; POSIX-fd/fabric handles)"),
            },
            "gbs_per_pair": round(total / pairs / t_dev / 1e9, 2),
            # loopback never touches NVLink: no link fraction there
            "frac_of_nvlink_900_per_pair": (round(total / pairs / t_dev / 1e9 /
                                                  NVLINK_NOMINAL_GBS, 4) if multi else None),
            "p50_latency_ms": round(nearest_rank(lat_req, 50) / 1e6, 4),
            "p90_latency_ms": round(nearest_rank(lat_req, 90) / 1e6, 4),
            "latency": {
                "what": ("isolated requests: host wall from kvd_pull entry to kvd_wait_done "
                         "observing the completion word, one request at a time on an idle pair, "
                         "all pairs starting each request together"
                         + ("; per request the MAX over the TP-shard ranks"
                            if args.config == "c4" and len(dec) > 1 else "")),
                "requests_timed": len(lat_req),
                "per_pair_pooled_p50_ms": round(nearest_rank(lat_all, 50) / 1e6, 4),
                "queued_p50_ms": (round(nearest_rank([x for s in dec for x in s["lat_queued"]],
                                                     50) / 1e6, 4)
                                  if dec[0]["lat_queued"] else None),
                "queued_p90_ms": (round(nearest_rank([x for s in dec for x in s["lat_queued"]],
                                                     90) / 1e6, 4)
                                  if dec[0]["lat_queued"] else None),
                "queued_what": ("the pair's requests issued together as in a timed step, "
                                "issue -> completion observed (includes queueing)")
                               if dec[0]["lat_queued"] else None,
                "engine_p50_ms": (round(nearest_rank(engine_req, 50) / 1e6, 4)
                                  if engine_req else None),
                "engine_p90_ms": (round(nearest_rank(engine_req, 90) / 1e6, 4)
                                  if engine_req else None),
                "engine_what": (f"--engine {args.engine}: the same isolated requests posted to "
                                "the resident pull engine (KVD_OPT_ENGINE: no launch per "
                                "request; requests > 2 MiB still launch)")
                               if engine_req else None},
            "step_device_ms": round(step_dev, 4),
            "kernel_ms_per_step": round(kern_dev, 4),
            "roofline": roof,
            "e2e": {"value": round(total / t_wall / 1e9, 2), "unit": "GB/s",
                    "h2d_bytes_per_step": 8 * n_blocks * pairs, "d2h_bytes_per_step": 8 * n_req * pairs,
                    "what": "host wall from kvd_pull entry (host block-id tables -> kernel "
                            "parameters) to the host observing the pinned completion words"},
            "gpu_launches": sum(s["launches"] for s in dec),
            "calibration": {
                "copy_engine_gbs_per_pair": (round(float(np.mean([s["ce_gbs"] for s in dec])), 1)
                                             if all(s["ce_gbs"] for s in dec) else None),
                "mover_contiguous_gbs_per_pair": (
                    round(float(np.mean([s["tma_gbs"] for s in dec])), 1)
                    if all(s["tma_gbs"] for s in dec) else None),
                "what": "a contiguous request as large as the first request of a step over the "
                        "same mapping: (copy engine) one cudaMemcpyAsync per (layer, K/V) "
                        "segment; (tma) the product's own mover and launch policy -- how much "
                        "the fragmented block table costs"},
            "parity": bool(all(oks)),
            "clocks": clk,
        }
        if multi and not args.no_nccl:
            nb_out = {}
            names = sorted({k for s_ in all_stats if s_["base"] for k in s_["base"]})
            for name in names:
                rs = [s_["base"][name] for s_ in all_stats
                      if s_["base"] and name in s_["base"] and s_["base"][name]["bytes"]]
                if not rs:
                    continue
                t = max(r["wall_s"] for r in rs)
                tot = sum(r["bytes"] for r in rs)
                lat = [x for r in rs for x in r["lat"]]
                oks_b = [s_["base"][name]["ok"] for s_ in all_stats
                         if s_["base"] and name in s_["base"]]
                nb_out[name] = {"value": round(tot / t / 1e9, 2), "unit": "GB/s",
                                "gbs_per_pair": round(tot / pairs / t / 1e9, 2),
                                "p50_step_latency_ms": round(nearest_rank(lat, 50) * 1e3, 4),
                                "steps": rs[0]["steps"], "messages_per_step": rs[0]["segments"],
                                "parity": bool(all(oks_b))}
            transfers = {k: v for k, v in nb_out.items() if not k.startswith("n0")}
            best = max(transfers, key=lambda k: transfers[k]["value"])
            nb_out["best_transfer"] = best
            nb_out["kvd_pull_vs_best_transfer"] = round(out["value"] / nb_out[best]["value"], 3)
            nb_out["kvd_pull_e2e_vs_best_transfer"] = round(
                out["e2e"]["value"] / nb_out[best]["value"], 3)
            if "n0_raw_contiguous" in nb_out:
                nb_out["kvd_pull_vs_n0_link_ceiling"] = round(
                    out["value"] / nb_out["n0_raw_contiguous"]["value"], 3)
            nb_out["what"] = ("NCCL 2.28 send/recv via torch.distributed on the same caches and "
                              "block tables; host wall per step incl. the block-id message "
                              "(N1 whole request staged; N2 one message per segment; N3 "
                              "double-buffered chunks; N0 one contiguous message of the same "
                              "bytes, no paged layout = NCCL's link ceiling)")
            out["nccl_baseline"] = nb_out
        if not multi and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_oracle_sample()
        else:   # the contract times the oracle on rank 0 at N = 1 only
            out["cpu_baseline"] = None
        print(json.dumps(out), flush=True)

    if peer:
        peer.close()
    if multi:
        dist.barrier(group=gloo)
    for c in (dst, src):
        if c:
            c.close()


def main():
    ap = argparse.ArgumentParser(description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["kvd", "reference"], default="kvd")
    ap.add_argument("--config", choices=["c1", "c2", "c3", "c4"], default="c2")
    ap.add_argument("--table", choices=["fragmented", "contiguous", "worst"], default="fragmented")
    ap.add_argument("--batch", action="store_true",
                    help="issue each step's requests with one kvd_pull_batch (f1)")
    ap.add_argument("--variant", choices=["lsu", "lsu32", "ce", "tma"], default=None,
                    help="default: library auto (TMA ring over NVLink, LSU in loopback)")
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--max-ctas", type=int, default=0)
    ap.add_argument("--no-coalesce", action="store_true")
    ap.add_argument("--timing", choices=["timer", "events"], default="timer",
                    help="roofline timing: region events + in-kernel globaltimer (default) or "
                         "library events around every launch")
    ap.add_argument("--streams", type=int, default=0,
                    help="KVD_OPT_STREAMS: >= 2 lets consecutive pulls overlap on library "
                         "streams (completion still polled per request)")
    ap.add_argument("--early", type=int, default=None,
                    help="KVD_OPT_EARLY_LOADS (ring stages read before the preceding pull ends)")
    ap.add_argument("--pairing", choices=["rail", "ring"], default="rail",
                    help="rail (default): ranks [0, N/2) prefill, rank k -> N/2 + k; ring: a "
                         "stress of the switch -- every rank holds both caches and pulls from "
                         "rank k+1 mod N (N concurrent pulls; no NCCL comparators)")
    ap.add_argument("--memory", choices=["torch", "vmm"], default="torch",
                    help="cache memory: torch/cudaMalloc (legacy IPC) or kvd_mem_alloc (VMM, "
                         "POSIX-fd/fabric handles, §8 f3 groundwork)")
    ap.add_argument("--engine", type=int, default=0,
                    help="also time the isolated-request latency through the resident pull "
                         "engine with this many CTAs (KVD_OPT_ENGINE)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nccl", action="store_true", help="skip the NCCL send/recv baselines")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # the NCCL baselines' send/recv are serialised by design (one pair)
        os.environ.setdefault("TORCH_NCCL_SHOW_EAGER_INIT_P2P_SERIALIZATION_WARNING", "false")
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        if world % 2:
            raise SystemExit("N > 1 must be even (prefill/decode pairs)")
    run_kvd(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
