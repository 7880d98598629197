# ncu --set full (+ NVLink counters) of the final kernel over NVLink: the C2
# and C4 pulls (auto policy) and the C2 push, one launch each, GPU0 -> GPU1.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
NV="nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvlrx__bytes_data_protocol.sum,nvlrx__bytes_packet_response_data_user.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes_packet_request_data_protocol.sum,nvltx__bytes_data_protocol.sum"
for c in c2 c4; do
  Q="python tools/sweep.py --src-dev 0 --dst-dev 1 --profile-once --variants auto --config $c"
  $Q > gpurun_out/r02n_plain_$c.log 2>&1 && timeout 600 ncu --set full --metrics $NV --clock-control none --import-source on -k regex:pull_kernel -s 1 -c 1 -o gpurun_out/r02n_prof_nvlink_$c $Q > gpurun_out/r02n_ncu_$c.log 2>&1; echo PROF_$c $?
done
Q="python tools/sweep.py --src-dev 0 --dst-dev 1 --profile-once --variants auto --config c2 --mode push"
$Q > gpurun_out/r02n_plain_push.log 2>&1 && timeout 600 ncu --set full --metrics $NV --clock-control none --import-source on -k regex:pull_kernel -s 1 -c 1 -o gpurun_out/r02n_prof_nvlink_push $Q > gpurun_out/r02n_ncu_push.log 2>&1; echo PROF_push $?
ls -la gpurun_out/ | grep r02n_prof
