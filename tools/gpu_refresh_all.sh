# Round-1 refresh on a 4-GPU box: GPU tests, bench lines N = 1/2/4 (C1-C4),
# the reference arm, and the N = 1 launch list + ncu capture (single process).
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r_tests.log 2>&1; echo TESTS $?; tail -2 gpurun_out/r_tests.log
python bench.py --steps 50 --warmup 5 > gpurun_out/r_n1.log 2>&1; echo N1 $?
T="timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
$T --nproc-per-node 2 --master-port 29701 bench.py --gpus 2 --steps 50 --warmup 5 > gpurun_out/r_n2.log 2>&1; echo N2 $?
$T --nproc-per-node 4 --master-port 29702 bench.py --gpus 4 --steps 50 --warmup 5 > gpurun_out/r_n4.log 2>&1; echo N4 $?
$T --nproc-per-node 4 --master-port 29703 bench.py --gpus 4 --config c3 --steps 5 --warmup 3 > gpurun_out/r_n4_c3.log 2>&1; echo N4C3 $?
$T --nproc-per-node 4 --master-port 29704 bench.py --gpus 4 --config c3 --batch --steps 5 --warmup 3 --no-nccl > gpurun_out/r_n4_c3b.log 2>&1; echo N4C3B $?
$T --nproc-per-node 4 --master-port 29705 bench.py --gpus 4 --config c4 --steps 50 --warmup 5 > gpurun_out/r_n4_c4.log 2>&1; echo N4C4 $?
$T --nproc-per-node 2 --master-port 29706 bench.py --gpus 2 --config c1 --steps 200 --warmup 10 --no-nccl > gpurun_out/r_n2_c1.log 2>&1; echo N2C1 $?
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r_ref.log 2>&1; echo REF $?
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/r_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r_launches_n1.csv $B > gpurun_out/r_ncu1.log 2>&1; echo LAUNCH $?
$B > gpurun_out/r_plain2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 3 -c 1 -o gpurun_out/r_prof_n1 $B > gpurun_out/r_ncu2.log 2>&1; echo PROF $?
for f in r_n1 r_n2 r_n4 r_n4_c3 r_n4_c3b r_n4_c4 r_n2_c1 r_ref; do grep '^{' gpurun_out/$f.log > gpurun_out/$f.json; done
