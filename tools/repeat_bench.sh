# Run-to-run spread of the headline lines: 5 x N=2 C2 and 5 x N=1 loopback C2
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
for i in 1 2 3 4 5; do
  $T --master-port $((29990+i)) bench.py --gpus 2 --steps 30 --warmup 5 --no-nccl --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'n': 2, 'run': $i, 'value': d['value'], 'kernel': d['roofline']['achieved'], 'gt': d['roofline'].get('globaltimer_cross_check',{}).get('achieved'), 'clk': d['clocks']['sm_mhz']}))"
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'n': 1, 'run': $i, 'value': d['value'], 'kernel': d['roofline']['achieved'], 'frac': d['roofline']['frac'], 'clk': d['clocks']['sm_mhz']}))"
done
