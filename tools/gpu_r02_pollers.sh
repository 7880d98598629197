# 2-GPU box: engine pollers A/B (1 / 2 / 4 staggered polling warps), C1 over NVLink and loopback
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
OUT=gpurun_out/r02_engine_pollers.jsonl; : > $OUT
export KVD_LAT_C1_ONLY=1
for np in 1 2 4; do
  if [ $np = 1 ]; then bash tools/build_variant.sh pollers1 > /dev/null; else sed "s/kPollers = 4;/kPollers = $np;/" tools/ab_patches/engine_pollers4.patch > paper_2501_14743_b200/ab/p$np.patch; bash tools/build_patched.sh pollers$np paper_2501_14743_b200/ab/p$np.patch > /dev/null; fi
  D=$PWD/paper_2501_14743_b200/ab/pollers$np
  nvcc -O2 -I include tools/native/kvd_latency.cu -L $D -lkvd -Xlinker -rpath=$D -o $D/kvd_latency 2>/dev/null
  for rep in 1 2; do
    for e in 8 16; do
      echo "{\"pollers\": $np, \"rep\": $rep}" >> $OUT
      timeout 120 $D/kvd_latency 0 1 2000 0 $e >> $OUT 2>&1
      timeout 120 $D/kvd_latency 0 1 2000 1 $e >> $OUT 2>&1
    done
  done
  timeout 120 $D/kvd_latency 0 0 2000 0 8 >> $OUT 2>&1
done
python - <<'PY'
import json
p=None
for l in open("gpurun_out/r02_engine_pollers.jsonl"):
    d=json.loads(l)
    if "pollers" in d: p=d["pollers"]; continue
    print(p, d["src_dev"], d["dst_dev"], d["ctas"], d["latency_us_p50"], d["latency_us_min"], d["kernel_span_us_p50"], d["pre_us_p50"])
PY
