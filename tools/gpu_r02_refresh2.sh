# final refresh with the final kernel, 2-GPU box: bench lines + C5 sweep
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T="timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29711 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02q_n2_c2.log 2>&1; echo N2C2 $?
$T --master-port 29712 bench.py --gpus 2 --steps 20 --warmup 5 --config c4 > gpurun_out/r02q_n2_c4.log 2>&1; echo N2C4 $?
$T --master-port 29713 bench.py --gpus 2 --steps 100 --warmup 5 --config c1 --engine 8 > gpurun_out/r02q_n2_c1.log 2>&1; echo N2C1 $?
$T --master-port 29714 bench.py --gpus 2 --steps 5 --warmup 3 --config c3 > gpurun_out/r02q_n2_c3.log 2>&1; echo N2C3 $?
$T --master-port 29715 bench.py --gpus 2 --steps 5 --warmup 3 --config c3 --batch --no-nccl > gpurun_out/r02q_n2_c3b.log 2>&1; echo N2C3B $?
$T --master-port 29716 tools/c5_sweep.py --iters 10 > gpurun_out/r02q_c5_sweep_n2.jsonl 2> gpurun_out/r02q_c5_err.log; echo C5 $?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02q_n1.log 2>&1; echo N1 $?
for f in r02q_n1 r02q_n2_c2 r02q_n2_c4 r02q_n2_c1 r02q_n2_c3 r02q_n2_c3b; do grep '^{' gpurun_out/$f.log | cut -c1-200; done
