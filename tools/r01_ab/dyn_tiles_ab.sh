python -m pytest -q tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_batch.py tests/test_gpu_release.py tests/test_gpu_policy.py > gpurun_out/t20.log 2>&1; tail -1 gpurun_out/t20.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
for lib in "" "KVD_LIB_PATH=$PWD/paper_2501_14743_b200/ab/static/libkvd.so"; do
  for c in c4 c2; do
    env $lib $T --master-port 29951 bench.py --gpus 2 --config $c --steps 30 --warmup 3 --no-nccl --no-cpu-baseline > gpurun_out/dyn.log 2>&1
    grep "^{" gpurun_out/dyn.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib'[-20:], '$c', d['value'], d['roofline']['achieved'], d['roofline'].get('globaltimer_cross_check',{}).get('achieved'))"
  done
done
