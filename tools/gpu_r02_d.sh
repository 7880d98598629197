# round 2: early-load depth sweep (ring stages read before the wait) and
# library streams for back-to-back short pulls.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
TL="timeout 600 python tools/timeline.py --config c4 --tokens 128,1024 --requests 24"
for e in 0 1 2 3 4 8 0 2 8; do $TL --early $e --label depth$e >> gpurun_out/r02d_tl.jsonl 2>>gpurun_out/r02d_err.log; done
timeout 600 python tools/small_requests.py --config c4 --tokens 128,1024 --requests 24 --modes single,lib2,batch --timing 0 >> gpurun_out/r02d_small.jsonl 2>>gpurun_out/r02d_err.log
python -c "
import json
for l in open('gpurun_out/r02d_tl.jsonl'):
    d=json.loads(l); print(d['label'], d['tokens'], d['us_median'], 'period GB/s', d['gbs_per_period'])
for l in open('gpurun_out/r02d_small.jsonl'):
    d=json.loads(l); print(d['tokens_per_request'], {k: v for k, v in d.items() if k.endswith('_gbs')})
"
tail -3 gpurun_out/r02d_err.log
