#!/usr/bin/env python
"""Check bench.py JSON lines against the benchmark contract's required keys.

    python tools/check_bench_line.py profiles/r01_final_*.json
"""
import json
import sys

TOP = {"metric": str, "value": (int, float), "unit": str, "n_gpus": int, "steps": int,
       "warmup": int, "ms_per_step": (int, float), "higher_is_better": bool, "scaling": str,
       "dtype": str, "data": str, "config": dict, "e2e": dict, "gpu_launches": int,
       "clocks": dict}
KVD = {"roofline": dict, "cpu_baseline": dict}
ROOF = {"bound", "achieved", "peak", "unit", "frac", "traffic"}
E2E = {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"}
CLK = {"sm_mhz", "sm_max_mhz", "reasons"}
BAD_REASONS = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}


def check(d):
    errs = []
    ref = d.get("impl") == "reference"
    for k, t in TOP.items():
        if ref and k in ("clocks", "gpu_launches"):
            continue
        if k not in d:
            errs.append(f"missing {k}")
        elif not isinstance(d[k], t):
            errs.append(f"{k} has type {type(d[k]).__name__}")
    if "workload" not in d.get("config", {}):
        errs.append("config.workload missing")
    if not E2E <= set(d.get("e2e", {})):
        errs.append(f"e2e lacks {E2E - set(d.get('e2e', {}))}")
    if not ref:
        for k in KVD:
            if k not in d:
                errs.append(f"missing {k}")
        if d.get("n_gpus") == 1 and not d.get("cpu_baseline"):
            errs.append("N = 1 line without a cpu_baseline")
        roof = d.get("roofline", {})
        if not ROOF <= set(roof):
            errs.append(f"roofline lacks {ROOF - set(roof)}")
        if roof and roof.get("peak") and abs(roof["achieved"] / roof["peak"] - roof["frac"]) > 1e-3:
            errs.append("roofline.frac != achieved / peak")
        clk = d.get("clocks", {})
        if not CLK <= set(clk):
            errs.append(f"clocks lacks {CLK - set(clk)}")
        if BAD_REASONS & set(clk.get("reasons", [])):
            errs.append(f"throttled: {clk['reasons']}")
        if d.get("gpu_launches", 0) <= 0:
            errs.append("gpu_launches <= 0")
        if d.get("warmup", 0) < 3:
            errs.append("warmup < 3")
        cb = d.get("cpu_baseline")
        if d.get("n_gpus") == 1 and cb:
            for k in ("value", "unit", "cores", "kind", "sample"):
                if k not in cb:
                    errs.append(f"cpu_baseline lacks {k}")
    else:
        if "cpu_baseline" not in d:
            errs.append("reference line lacks cpu_baseline")
    return errs


def main(paths):
    bad = 0
    for p in paths:
        for line in open(p):
            line = line.strip()
            if not line.startswith("{"):
                continue
            errs = check(json.loads(line))
            print(("OK   " if not errs else "FAIL ") + p + ("" if not errs else ": " + "; ".join(errs)))
            bad += bool(errs)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
