# ncu evidence for the current kernels (one tool per call: ncu only)
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/p_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches_n1.csv $B > gpurun_out/p_ncu1.log 2>&1; echo LAUNCH $?
$B > gpurun_out/p_plain2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 3 -c 1 -o gpurun_out/p_prof_n1 $B > gpurun_out/p_ncu2.log 2>&1; echo PROF1 $?
Q="python tools/sweep.py --src-dev 0 --dst-dev 1 --profile-once --variants tma --threads 32 --stages 6 --tiles 32768 --ctas 32"
$Q > gpurun_out/p_plain3.log 2>&1 && timeout 600 ncu --set full --metrics nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvlrx__bytes_data_protocol.sum,nvlrx__bytes_packet_response_data_user.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes_packet_request_data_protocol.sum --clock-control none --import-source on -k regex:pull_kernel -s 1 -c 1 -o gpurun_out/p_prof_nvlink $Q > gpurun_out/p_ncu3.log 2>&1; echo PROF2 $?
