# --streams 2 under the default (region-event) roofline timing
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
for st in 0 2; do
  for c in c4 c2 c3; do
    $T --master-port 29987 bench.py --gpus 2 --config $c --steps 20 --warmup 3 --no-nccl --no-cpu-baseline --streams $st > gpurun_out/sta.log 2>&1
    grep "^{" gpurun_out/sta.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(json.dumps({'streams': $st, 'config': '$c', 'value': d['value'], 'achieved': r['achieved'], 'frac': r['frac'], 'parity': d['parity']}))"
  done
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --streams $st 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(json.dumps({'streams': $st, 'config': 'n1', 'value': d['value'], 'achieved': r['achieved'], 'frac': r['frac'], 'parity': d['parity']}))"
done
