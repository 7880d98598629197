mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for lib in base claim4; do
  L=""; [ $lib != base ] && L="KVD_LIB_PATH=$PWD/paper_2501_14743_b200/ab/$lib/libkvd.so"
  env $L timeout 600 python tools/timeline.py --config c4 --tokens 128,1024,8192 --requests 24 --early 2 --label $lib >> gpurun_out/r02m_tl.jsonl 2>> gpurun_out/r02m_err.log
  env $L timeout 600 python tools/timeline.py --config c2 --tokens 128,8192 --requests 12 --early 2 --label $lib >> gpurun_out/r02m_tl.jsonl 2>> gpurun_out/r02m_err.log
done
python -c "
import json
for l in open('gpurun_out/r02m_tl.jsonl'):
    d=json.loads(l); print(d['label'], d['config'], d['tokens'], d['us_median'], 'period GB/s', d['gbs_per_period'])
"
