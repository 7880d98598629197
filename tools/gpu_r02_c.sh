# round 2: what stretches the hand-off between back-to-back pulls (A/B patches
# in tools/ab_patches/, timing only) and ring-size variants with early loads.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
TL="timeout 600 python tools/timeline.py --config c4 --tokens 128,1024 --requests 24"
for e in 1 0; do
  $TL --early $e --label base >> gpurun_out/r02c_tl.jsonl 2>>gpurun_out/r02c_err.log
  for ab in relaxed_flag late_trigger; do
    KVD_LIB_PATH=$PWD/paper_2501_14743_b200/ab/$ab/libkvd.so $TL --early $e --label $ab >> gpurun_out/r02c_tl.jsonl 2>>gpurun_out/r02c_err.log
  done
done
for st in 2 3 4; do $TL --early 1 --stages $st --label stages$st >> gpurun_out/r02c_tl.jsonl 2>>gpurun_out/r02c_err.log; done
for c in 24 32 96; do $TL --early 1 --ctas $c --label ctas$c >> gpurun_out/r02c_tl.jsonl 2>>gpurun_out/r02c_err.log; done
python -c "
import json
for l in open('gpurun_out/r02c_tl.jsonl'):
    d=json.loads(l); print(d['label'], d['tokens'], 'early', d['early'], d['us_median'], 'period GB/s', d['gbs_per_period'], d['info']['ctas'])
"
tail -3 gpurun_out/r02c_err.log
