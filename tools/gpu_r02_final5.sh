# round 2 closing run on a 2-GPU box: the whole GPU suite (fuzz and stress
# included) and the C1 bench line with the faster binding.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02z_smoke.log 2>&1; echo SMOKE $?
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/r02z_tests_2gpu.log 2>&1; echo TESTS $?; tail -4 gpurun_out/r02z_tests_2gpu.log
T="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29981 bench.py --gpus 2 --steps 100 --warmup 5 --config c1 --engine 16 > gpurun_out/r02z_n2_c1.log 2>&1; echo N2C1 $?
grep '^{' gpurun_out/r02z_n2_c1.log | cut -c1-200
