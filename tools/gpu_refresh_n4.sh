# Full refresh on a 4-GPU box: tests, bench lines at N = 1/2/4, C3/C4, C5 sweep at 2 pairs
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r_tests.log 2>&1; echo TESTS $?; tail -2 gpurun_out/r_tests.log
python bench.py --steps 50 --warmup 5 > gpurun_out/r_n1.log 2>&1; echo N1 $?
T="timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
$T --nproc-per-node 2 --master-port 29701 bench.py --gpus 2 --steps 50 --warmup 5 > gpurun_out/r_n2.log 2>&1; echo N2 $?
$T --nproc-per-node 4 --master-port 29702 bench.py --gpus 4 --steps 50 --warmup 5 > gpurun_out/r_n4.log 2>&1; echo N4 $?
$T --nproc-per-node 4 --master-port 29703 bench.py --gpus 4 --config c3 --steps 5 --warmup 3 > gpurun_out/r_n4_c3.log 2>&1; echo N4C3 $?
$T --nproc-per-node 4 --master-port 29704 bench.py --gpus 4 --config c3 --batch --steps 5 --warmup 3 --no-nccl > gpurun_out/r_n4_c3b.log 2>&1; echo N4C3B $?
$T --nproc-per-node 4 --master-port 29705 bench.py --gpus 4 --config c4 --steps 50 --warmup 5 > gpurun_out/r_n4_c4.log 2>&1; echo N4C4 $?
$T --nproc-per-node 2 --master-port 29706 bench.py --gpus 2 --config c1 --steps 200 --warmup 10 --no-nccl > gpurun_out/r_n2_c1.log 2>&1; echo N2C1 $?
$T --nproc-per-node 4 --master-port 29707 tools/c5_sweep.py --iters 10 > gpurun_out/r_c5_n4.jsonl 2> gpurun_out/r_c5_n4.err; echo C5 $?
for f in r_n1 r_n2 r_n4 r_n4_c3 r_n4_c3b r_n4_c4 r_n2_c1; do grep '^{' gpurun_out/$f.log > gpurun_out/$f.json; done
