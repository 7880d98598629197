set -x
python bench.py --steps 30 --warmup 5 > gpurun_out/b_n1_c2.log 2>&1; echo N1 $?
T="timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
$T --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 --steps 30 --warmup 5 > gpurun_out/b_n2_c2.log 2>&1; echo N2 $?
$T --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 --steps 30 --warmup 5 > gpurun_out/b_n4_c2.log 2>&1; echo N4 $?
$T --nproc-per-node 4 --master-port 29603 bench.py --gpus 4 --config c3 --steps 5 --warmup 3 > gpurun_out/b_n4_c3.log 2>&1; echo N4C3 $?
$T --nproc-per-node 4 --master-port 29604 bench.py --gpus 4 --config c3 --batch --steps 5 --warmup 3 --no-nccl > gpurun_out/b_n4_c3_batch.log 2>&1; echo N4C3B $?
$T --nproc-per-node 4 --master-port 29605 bench.py --gpus 4 --config c4 --steps 50 --warmup 5 > gpurun_out/b_n4_c4.log 2>&1; echo N4C4 $?
$T --nproc-per-node 2 --master-port 29606 bench.py --gpus 2 --config c1 --steps 200 --warmup 10 --no-nccl > gpurun_out/b_n2_c1.log 2>&1; echo N2C1 $?
P="python tools/sweep.py --src-dev 0 --dst-dev 1 --profile-once --variants tma --threads 32 --stages 6 --tiles 32768 --ctas 32"
$P > gpurun_out/plain_tma.log 2>&1 && timeout 600 ncu --set full --metrics nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvlrx__bytes_data_protocol.sum,nvlrx__bytes_packet_response_data_user.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes_packet_request_data_protocol.sum --clock-control none --import-source on -k regex:pull_kernel -s 1 -c 1 -o gpurun_out/prof_c2_nvlink_tma $P > gpurun_out/ncu_tma.log 2>&1; echo PROF $?
for f in gpurun_out/b_*.log; do echo "== $f"; grep '^{' $f | cut -c1-200; done
