# round 2: N = 2 bench lines with the one-launch link calibration (the NVLink
# roofline's peak), after tools/gpu_r02_final3.sh (whose N = 1 / reference
# lines stand: nothing on their path changed since).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T="timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29871 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02m_n2_c2.log 2>&1; echo N2C2 $?
$T --master-port 29872 bench.py --gpus 2 --steps 20 --warmup 5 --config c4 > gpurun_out/r02m_n2_c4.log 2>&1; echo N2C4 $?
$T --master-port 29873 bench.py --gpus 2 --steps 100 --warmup 5 --config c1 --engine 16 > gpurun_out/r02m_n2_c1.log 2>&1; echo N2C1 $?
$T --master-port 29874 bench.py --gpus 2 --steps 5 --warmup 3 --config c3 > gpurun_out/r02m_n2_c3.log 2>&1; echo N2C3 $?
$T --master-port 29875 bench.py --gpus 2 --steps 5 --warmup 3 --config c3 --batch --no-nccl > gpurun_out/r02m_n2_c3b.log 2>&1; echo N2C3B $?
for f in r02m_n2_c2 r02m_n2_c4 r02m_n2_c1 r02m_n2_c3 r02m_n2_c3b; do grep '^{' gpurun_out/$f.log | cut -c1-200; done
