# A/B: bulk L2 prefetch of the first ring before griddepcontrol.wait
# (tools/ab_patches/early_prefetch_l2.patch) vs the product, back-to-back C4 shards
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/build_patched.sh prefetch tools/ab_patches/early_prefetch_l2.patch > /dev/null
OUT=gpurun_out/r02_prefetch_ab.jsonl; : > $OUT
TL="timeout 300 python tools/timeline.py --config c4 --tokens 128,1024,8192 --requests 24"
for rep in 1 2; do
  for e in 2 0; do
    $TL --early $e --label base >> $OUT 2>>gpurun_out/r02_prefetch.err
    KVD_LIB_PATH=$PWD/paper_2501_14743_b200/ab/prefetch/libkvd.so $TL --early $e --label prefetch >> $OUT 2>>gpurun_out/r02_prefetch.err
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/r02_prefetch_ab.jsonl"):
    d = json.loads(l); m = d["us_median"]
    print(f'{d["label"]:9s} e{d["early"]} {d["tokens"]:5d} ctas={d["info"]["ctas"]:3d} per={d["gbs_per_period"]:6.1f} span={m["span"]:7.2f} pre={m["pre"]:5.2f} period={m["period"]:7.2f} handoff={m["handoff"]:5.2f}')
PY
tail -3 gpurun_out/r02_prefetch.err
