# bench timing modes: --timing timer (default: region events + in-kernel globaltimer) vs events
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
for tm in timer events; do
  for c in c4 c2 c3; do
    $T --master-port 29985 bench.py --gpus 2 --config $c --steps 20 --warmup 3 --no-nccl --no-cpu-baseline --timing $tm > gpurun_out/tab.log 2>&1
    grep "^{" gpurun_out/tab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(json.dumps({'timing': '$tm', 'config': '$c', 'value': d['value'], 'achieved': r['achieved'], 'frac': r['frac'], 'gt': r.get('globaltimer_cross_check',{}).get('achieved')}))"
  done
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --timing $tm 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(json.dumps({'timing': '$tm', 'config': 'n1', 'value': d['value'], 'achieved': r['achieved'], 'frac': r['frac'], 'gt': r.get('globaltimer_cross_check',{}).get('achieved')}))"
done
