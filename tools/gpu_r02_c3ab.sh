mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for rep in 1 2; do
for lib in base claim2_always; do
  L=""; [ $lib != base ] && L="KVD_LIB_PATH=$PWD/paper_2501_14743_b200/ab/$lib/libkvd.so"
  for c in c3 c4 c2; do
  env $L $T --master-port 29721 bench.py --gpus 2 --config $c --steps 5 --warmup 3 --no-nccl > gpurun_out/c3ab.log 2>&1
  grep '^{' gpurun_out/c3ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'$lib','config':'$c','rep':$rep,'value':d['value'],'gt':d['roofline'].get('globaltimer_cross_check',{}).get('achieved')}))" >> gpurun_out/r02r_c3ab.jsonl
  done
done
done
cat gpurun_out/r02r_c3ab.jsonl
