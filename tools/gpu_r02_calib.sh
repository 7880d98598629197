# 2-GPU box: the link calibration kernel (kvd_peer_calibrate) -- its tests,
# and the bench lines whose NVLink roofline now divides by it.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02c_build.log 2>&1; echo BUILD $?
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_gpu_policy.py tests/test_abi_host.py -rs > gpurun_out/r02c_tests.log 2>&1; echo TESTS $?; tail -3 gpurun_out/r02c_tests.log
T="timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29681 bench.py --gpus 2 --steps 20 --warmup 5 --no-nccl > gpurun_out/r02c_n2_c2.log 2>&1; echo N2C2 $?
$T --master-port 29682 bench.py --gpus 2 --steps 20 --warmup 5 --no-nccl --config c4 > gpurun_out/r02c_n2_c4.log 2>&1; echo N2C4 $?
for f in r02c_n2_c2 r02c_n2_c4; do grep '^{' gpurun_out/$f.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['value'], r['achieved'], r['peak'], r['frac'], r['frac_of_read_user_ceiling_800'], json.dumps(r['measured_read_ceiling']))"; tail -3 gpurun_out/$f.log | cut -c1-300; done
