#!/usr/bin/env python
"""Summarise ncu output for profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py launches <launches.csv>          -> per-kernel share table
  python tools/ncu_summary.py report <x.ncu-rep> <out.json> [bytes_per_launch]
"""
import csv
import io
import json
import subprocess
import sys

UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
        "second": 1e6, "s": 1e6}
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "nvlrx__bytes.sum", "nvlrx__bytes_data_user.sum",
        "nvlrx__bytes_data_protocol.sum", "nvlrx__bytes_packet_response_data_user.sum",
        "nvltx__bytes.sum", "nvltx__bytes_data_user.sum",
        "nvltx__bytes_packet_request_data_protocol.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum",
        "launch__occupancy_limit_registers"]


def launches(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            h, start = r, i + 1
            break
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = {}
    for r in rows[start:]:
        if len(r) < len(h):
            continue
        us = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        tot.setdefault(r[ki].split("(")[0][:100], []).append(us)
    all_us = sum(sum(v) for v in tot.values())
    print("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -sum(x[1])):
        print(f"| `{k}` | {len(v)} | {sum(v):.1f} | {sum(v) / len(v):.1f} | "
              f"{sum(v) / all_us:.1%} |")


def report(path, out, alg=None):
    raw = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, v = rows[0], rows[1], rows[2]
    d = {}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            val = float(v[i].replace(",", ""))
            u = units[i]
            if u in BYTES:
                val *= BYTES[u]
                u = "byte"
            elif u in UNIT:
                val *= UNIT[u]
                u = "us"
            d[k] = {"value": val, "unit": u}
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else None
    res = {"report": path, "kernel": name, "metrics": d}
    rd = d.get("dram__bytes_read.sum", {}).get("value", 0)
    wr = d.get("dram__bytes_write.sum", {}).get("value", 0)
    res["dram_bytes_per_launch"] = rd + wr
    if alg:
        res["algorithmic_bytes_per_launch"] = int(alg)
        res["traffic_over_algorithmic"] = (rd + wr) / int(alg)
    t = d.get("gpu__time_duration.sum", {}).get("value")
    if t and "nvlrx__bytes_data_user.sum" in d:
        res["nvlink_rx_user_GBps"] = d["nvlrx__bytes_data_user.sum"]["value"] / t / 1e3
        res["nvlink_rx_total_GBps"] = d["nvlrx__bytes.sum"]["value"] / t / 1e3
        res["nvlink_rx_protocol_fraction"] = (d["nvlrx__bytes_data_protocol.sum"]["value"] /
                                              d["nvlrx__bytes.sum"]["value"])
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
