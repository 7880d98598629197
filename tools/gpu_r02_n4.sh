# round 2 on 4 GPUs: 2 rail pairs (C2, C3, C3 batched), 2 TP shard pairs (C4,
# request latency = max over shards), the GPU suite's 4-GPU tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T="timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29731 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02s_n4_c2.log 2>&1; echo N4C2 $?
$T --master-port 29732 bench.py --gpus 4 --steps 20 --warmup 5 --config c4 > gpurun_out/r02s_n4_c4.log 2>&1; echo N4C4 $?
$T --master-port 29733 bench.py --gpus 4 --steps 5 --warmup 3 --config c3 > gpurun_out/r02s_n4_c3.log 2>&1; echo N4C3 $?
$T --master-port 29734 bench.py --gpus 4 --steps 5 --warmup 3 --config c3 --batch --no-nccl > gpurun_out/r02s_n4_c3b.log 2>&1; echo N4C3B $?
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py -k "nvswitch" -rs > gpurun_out/r02s_tests.log 2>&1; echo TESTS $?
tail -3 gpurun_out/r02s_tests.log
for f in r02s_n4_c2 r02s_n4_c4 r02s_n4_c3 r02s_n4_c3b; do grep '^{' gpurun_out/$f.log | cut -c1-200; tail -2 gpurun_out/$f.log | cut -c1-300; done
timeout 1500 python -m pytest -q -p no:cacheprovider tests -m gpu -rs > gpurun_out/r02s_tests_4gpu.log 2>&1; echo TESTS4 $?; tail -3 gpurun_out/r02s_tests_4gpu.log
