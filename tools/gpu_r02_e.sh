# round 2: static first ring + claim-ahead; parity of the TMA paths; timeline.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_batch.py tests/test_gpu_heads.py tests/test_gpu_concurrency.py tests/test_gpu_release.py tests/test_gpu_policy.py -rs > gpurun_out/r02e_tests.log 2>&1; echo TESTS $?
tail -5 gpurun_out/r02e_tests.log
TL="timeout 600 python tools/timeline.py --config c4 --tokens 128,1024,8192 --requests 24"
for e in 0 2 8; do $TL --early $e --label claim_ahead_depth$e >> gpurun_out/r02e_tl.jsonl 2>>gpurun_out/r02e_err.log; done
timeout 600 python tools/timeline.py --config c2 --tokens 128,8192 --requests 12 --early 2 --label c2 >> gpurun_out/r02e_tl.jsonl 2>>gpurun_out/r02e_err.log
timeout 300 tools/native/kvd_latency 0 1 2000 1 > gpurun_out/r02e_lat01.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/r02e_tl.jsonl'):
    d=json.loads(l); print(d['label'], d['tokens'], d['us_median'], 'period GB/s', d['gbs_per_period'])
"
cat gpurun_out/r02e_lat01.jsonl
tail -3 gpurun_out/r02e_err.log
