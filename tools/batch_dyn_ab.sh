python -m pytest -q tests/test_gpu_batch.py tests/test_gpu_fuzz.py tests/test_gpu_release.py tests/test_gpu_vmm.py > gpurun_out/t28.log 2>&1; tail -1 gpurun_out/t28.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
for lib in "" "KVD_LIB_PATH=$PWD/paper_2501_14743_b200/ab/static/libkvd.so"; do
  env $lib $T --master-port 29991 bench.py --gpus 2 --config c3 --batch --steps 5 --warmup 3 --no-nccl --no-cpu-baseline > gpurun_out/bd.log 2>&1
  grep "^{" gpurun_out/bd.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('static' if '$lib' else 'dynamic', d['value'], d['parity'])"
done
