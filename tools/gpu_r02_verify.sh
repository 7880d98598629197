# adaptive claim size: bench C4 / C2 and the 10 MB timeline on one box
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for c in c4 c2; do
  $T --master-port 29692 bench.py --gpus 2 --config $c --steps 30 --warmup 5 --no-nccl > gpurun_out/v.log 2>&1
  grep '^{' gpurun_out/v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'config':'$c','value':d['value'],'gt':d['roofline'].get('globaltimer_cross_check',{}).get('achieved'),'p50':d['p50_latency_ms'],'parity':d['parity']}))" >> gpurun_out/r02n.jsonl
done
timeout 600 python tools/timeline.py --config c4 --tokens 128,1024,8192 --requests 24 --label adaptive >> gpurun_out/r02n_tl.jsonl 2>/dev/null
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x > gpurun_out/r02n_tests.log 2>&1; echo TESTS $?; tail -2 gpurun_out/r02n_tests.log
cat gpurun_out/r02n.jsonl
python -c "
import json
for l in open('gpurun_out/r02n_tl.jsonl'):
    d=json.loads(l); print(d['label'], d['config'], d['tokens'], d['us_median'], 'period GB/s', d['gbs_per_period'])
"
