"""The committed bench lines (profiles/r0[12]_final_*.json) satisfy the benchmark
contract's keys (tools/check_bench_line.py): metric/value/unit, roofline with
traffic, cpu_baseline at N = 1, e2e with host<->device bytes, gpu_launches,
clocks without throttle reasons, warm-up >= 3."""
import glob
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import check_bench_line  # noqa: E402

FILES = sorted(glob.glob(os.path.join(ROOT, "profiles", "r0[12]_final_*.json")))


@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(p) for p in FILES])
def test_committed_bench_line_meets_contract(path):
    lines = [l for l in open(path) if l.strip().startswith("{")]
    assert lines, path
    for l in lines:
        d = json.loads(l)
        assert check_bench_line.check(d) == [], path
        if d.get("impl") != "reference":
            assert d["parity"] is True
            assert d["roofline"]["unit"] == "GB/s" and d["roofline"]["peak"] > 0


def test_headline_lines_present():
    names = {os.path.basename(p) for p in FILES}
    assert {"r01_final_n1.json", "r01_final_n2.json", "r01_final_ref.json"} <= names
    assert {"r02_final_n1.json", "r02_final_n2_c2.json", "r02_final_ref.json"} <= names
