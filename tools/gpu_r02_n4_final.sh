# round 2 final evidence on a 4-GPU box: 2 rail pairs (C2, C3, C3 batched),
# 2 TP shard pairs (C4, request latency = max over shards), C1 (engine), the
# C5 sweep at 2 pairs, and the whole GPU suite (incl. the 4-GPU NVSwitch tests).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T="timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$T --master-port 29831 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02n4_c2.log 2>&1; echo N4C2 $?
$T --master-port 29832 bench.py --gpus 4 --steps 20 --warmup 5 --config c4 > gpurun_out/r02n4_c4.log 2>&1; echo N4C4 $?
$T --master-port 29833 bench.py --gpus 4 --steps 5 --warmup 3 --config c3 > gpurun_out/r02n4_c3.log 2>&1; echo N4C3 $?
$T --master-port 29834 bench.py --gpus 4 --steps 5 --warmup 3 --config c3 --batch --no-nccl > gpurun_out/r02n4_c3b.log 2>&1; echo N4C3B $?
$T --master-port 29835 bench.py --gpus 4 --steps 100 --warmup 5 --config c1 --engine 16 > gpurun_out/r02n4_c1.log 2>&1; echo N4C1 $?
for f in r02n4_c2 r02n4_c4 r02n4_c3 r02n4_c3b r02n4_c1; do grep '^{' gpurun_out/$f.log | cut -c1-200; done
timeout 1800 python -m pytest -q -p no:cacheprovider tests -m gpu -rs > gpurun_out/r02n4_tests.log 2>&1; echo TESTS4 $?; tail -3 gpurun_out/r02n4_tests.log
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29836 tools/c5_sweep.py --iters 10 > gpurun_out/r02_c5_sweep_n4.jsonl 2> gpurun_out/r02_c5n4_err.log; echo C5 $?
