# 2-GPU box: back-to-back short pulls (C4 shard, 128 / 1024 / 8192 tokens),
# launch-shape sweep with the %globaltimer timeline (tools/timeline.py).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
OUT=gpurun_out/r02_short_sweep.jsonl; : > $OUT
run() { timeout 300 python tools/timeline.py --config c4 --tokens 128,1024,8192 --requests 24 "$@" >> $OUT 2>>gpurun_out/r02_short_sweep.err; }
run --early 2 --label base
run --early 2 --ctas 64 --label ctas64
run --early 2 --ctas 96 --label ctas96
run --early 2 --ctas 148 --label ctas148
run --early 2 --tile 16384 --stages 8 --label t16s8
run --early 3 --label early3
run --early 1 --label early1
run --early 2 --stages 4 --label s4
run --early 2 --ctas 96 --stages 4 --label ctas96s4
run --early 2 --ctas 148 --stages 3 --label ctas148s3
run --early 2 --label base2
python - <<'PY'
import json
for l in open("gpurun_out/r02_short_sweep.jsonl"):
    d = json.loads(l); m = d["us_median"]
    print(f'{d["label"]:10s} {d["tokens"]:5d} ctas={d["info"]["ctas"]:3d} per={d["gbs_per_period"]:6.1f} span={m["span"]:7.2f} pre={m["pre"]:5.2f} period={m["period"]:7.2f} handoff={m["handoff"]:5.2f}')
PY
