# TMA ring at reduced grids (co-located decode): explicit 32/24/48 CTAs, early depth, claim variants
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for lib in base r01_claiming; do
  for c in 24 32 48; do
    for e in 0 2; do
      L=""; [ $lib != base ] && L="KVD_LIB_PATH=$PWD/paper_2501_14743_b200/ab/$lib/libkvd.so"
      env $L $T --master-port 29693 bench.py --gpus 2 --config c2 --steps 20 --warmup 5 --no-nccl --variant tma --threads 32 --stages 6 --tile 32768 --max-ctas $c --early $e > gpurun_out/ct.log 2>&1
      grep '^{' gpurun_out/ct.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'$lib','ctas':$c,'early':$e,'value':d['value'],'gt':d['roofline'].get('globaltimer_cross_check',{}).get('achieved')}))" >> gpurun_out/r02o_ctas.jsonl
    done
  done
done
cat gpurun_out/r02o_ctas.jsonl
