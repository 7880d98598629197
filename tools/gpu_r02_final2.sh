# round 2 final evidence on a 2-GPU box: bench lines (N=1, N=2 c1/c2/c3/c4),
# the reference arm, the ncu launch list of the N=1 bench, and ncu --set full
# captures of the pull kernel in loopback and over NVLink (C2, C4) and of push.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02j_n1.log 2>&1; echo N1 $?
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02j_ref.log 2>&1; echo REF $?
T="timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29671 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02j_n2_c2.log 2>&1; echo N2C2 $?
$T --master-port 29672 bench.py --gpus 2 --steps 20 --warmup 5 --config c4 > gpurun_out/r02j_n2_c4.log 2>&1; echo N2C4 $?
$T --master-port 29673 bench.py --gpus 2 --steps 100 --warmup 5 --config c1 --engine 8 > gpurun_out/r02j_n2_c1.log 2>&1; echo N2C1 $?
$T --master-port 29674 bench.py --gpus 2 --steps 5 --warmup 3 --config c3 > gpurun_out/r02j_n2_c3.log 2>&1; echo N2C3 $?
$T --master-port 29675 bench.py --gpus 2 --steps 5 --warmup 3 --config c3 --batch --no-nccl > gpurun_out/r02j_n2_c3b.log 2>&1; echo N2C3B $?
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/r02j_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02j_launches_n1.csv $B > gpurun_out/r02j_ncu1.log 2>&1; echo LAUNCH $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 3 -c 1 -o gpurun_out/r02j_prof_n1 $B > gpurun_out/r02j_ncu2.log 2>&1; echo PROF1 $?
NV="nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvlrx__bytes_data_protocol.sum,nvlrx__bytes_packet_response_data_user.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes_packet_request_data_protocol.sum,nvltx__bytes_data_protocol.sum"
for c in c2 c4; do
  Q="python tools/sweep.py --src-dev 0 --dst-dev 1 --profile-once --variants auto --config $c"
  $Q > gpurun_out/r02j_plain_$c.log 2>&1 && timeout 600 ncu --set full --metrics $NV --clock-control none --import-source on -k regex:pull_kernel -s 1 -c 1 -o gpurun_out/r02j_prof_nvlink_$c $Q > gpurun_out/r02j_ncu_$c.log 2>&1; echo PROF_$c $?
done
Q="python tools/sweep.py --src-dev 0 --dst-dev 1 --profile-once --variants auto --config c2 --mode push"
$Q > gpurun_out/r02j_plain_push.log 2>&1 && timeout 600 ncu --set full --metrics $NV --clock-control none --import-source on -k regex:pull_kernel -s 1 -c 1 -o gpurun_out/r02j_prof_nvlink_push $Q > gpurun_out/r02j_ncu_push.log 2>&1; echo PROF_push $?
for f in r02j_n1 r02j_ref r02j_n2_c2 r02j_n2_c4 r02j_n2_c1 r02j_n2_c3 r02j_n2_c3b; do grep '^{' gpurun_out/$f.log | cut -c1-250; done
ls -la gpurun_out/ | grep r02j
