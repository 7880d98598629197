# C4 A/B on one box: tile-claiming variants x early-read depth, through bench.py (N = 2)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for rep in 1 2; do
for lib in base claim4 r01_claiming; do
  for e in 0 2 8; do
    L=""; [ $lib != base ] && L="KVD_LIB_PATH=$PWD/paper_2501_14743_b200/ab/$lib/libkvd.so"
    env $L $T --master-port 29691 bench.py --gpus 2 --config c4 --steps 30 --warmup 5 --no-nccl --early $e > gpurun_out/c4ab.log 2>&1
    grep '^{' gpurun_out/c4ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'$lib','early':$e,'rep':$rep,'value':d['value'],'gt':d['roofline'].get('globaltimer_cross_check',{}).get('achieved'),'p50':d['p50_latency_ms']}))" >> gpurun_out/r02l_c4ab.jsonl
  done
done
done
cat gpurun_out/r02l_c4ab.jsonl
