# Programmatic dependent launch A/B: default build vs -DKVD_EXPERIMENT_NO_PDL
python -m pytest -q tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_batch.py tests/test_gpu_release.py tests/test_gpu_concurrency.py tests/test_gpu_heads.py > gpurun_out/t21.log 2>&1; tail -1 gpurun_out/t21.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
for lib in "" "KVD_LIB_PATH=$PWD/paper_2501_14743_b200/ab/nopdl/libkvd.so"; do
  for c in c4 c2; do
    env $lib $T --master-port 29971 bench.py --gpus 2 --config $c --steps 30 --warmup 3 --no-nccl --no-cpu-baseline > gpurun_out/pdl.log 2>&1
    grep "^{" gpurun_out/pdl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nopdl' if '$lib' else 'pdl', '$c', d['value'], d['roofline']['achieved'], d['roofline'].get('globaltimer_cross_check',{}).get('achieved'), d['p50_latency_ms'])"
  done
  env $lib python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/pdl1.log 2>&1
  grep "^{" gpurun_out/pdl1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nopdl' if '$lib' else 'pdl', 'n1', d['value'], d['roofline']['achieved'])"
  env $lib python tools/small_requests.py --ipc --config c4 --tokens 128,1024 --requests 16 --modes single 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('nopdl' if '$lib' else 'pdl', 'c4', d['tokens_per_request'], d['single_gbs'], d.get('single_step_us_per_request'), d.get('single_kernel_us_per_request'))"
done
