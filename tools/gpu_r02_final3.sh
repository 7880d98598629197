# round 2 final evidence (after the calibration kernel, the one-poller engine
# and the short-request grid) on a 2-GPU box: the GPU suite, bench lines
# (N=1, N=2 c1/c2/c3/c3-batched/c4), the reference arm, the short-request and
# timeline tables, the ncu launch list of the N=1 bench and ncu --set full of
# the loopback pull.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02k_smoke.log 2>&1; echo SMOKE $?
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/r02k_tests.log 2>&1; echo TESTS $?; tail -4 gpurun_out/r02k_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02k_n1.log 2>&1; echo N1 $?
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02k_ref.log 2>&1; echo REF $?
T="timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29771 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02k_n2_c2.log 2>&1; echo N2C2 $?
$T --master-port 29772 bench.py --gpus 2 --steps 20 --warmup 5 --config c4 > gpurun_out/r02k_n2_c4.log 2>&1; echo N2C4 $?
$T --master-port 29773 bench.py --gpus 2 --steps 100 --warmup 5 --config c1 --engine 16 > gpurun_out/r02k_n2_c1.log 2>&1; echo N2C1 $?
$T --master-port 29774 bench.py --gpus 2 --steps 5 --warmup 3 --config c3 > gpurun_out/r02k_n2_c3.log 2>&1; echo N2C3 $?
$T --master-port 29775 bench.py --gpus 2 --steps 5 --warmup 3 --config c3 --batch --no-nccl > gpurun_out/r02k_n2_c3b.log 2>&1; echo N2C3B $?
timeout 600 python tools/small_requests.py --ipc --config c4 --tokens 128,1024 --requests 16 > gpurun_out/r02k_small_c4.jsonl 2>gpurun_out/r02k_small.err; echo SMALL4 $?
timeout 600 python tools/small_requests.py --ipc --config c2 --tokens 128,512,4096 --requests 16 > gpurun_out/r02k_small_c2.jsonl 2>>gpurun_out/r02k_small.err; echo SMALL2 $?
timeout 600 python tools/timeline.py --config c4 --tokens 128,1024,8192 --requests 24 --early 2 --label final > gpurun_out/r02k_timeline.jsonl 2>>gpurun_out/r02k_small.err; echo TL $?
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/r02k_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02k_launches_n1.csv $B > gpurun_out/r02k_ncu1.log 2>&1; echo LAUNCH $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 3 -c 1 -o gpurun_out/r02k_prof_n1 $B > gpurun_out/r02k_ncu2.log 2>&1; echo PROF1 $?
for f in r02k_n1 r02k_ref r02k_n2_c2 r02k_n2_c4 r02k_n2_c1 r02k_n2_c3 r02k_n2_c3b; do grep '^{' gpurun_out/$f.log | cut -c1-200; done
