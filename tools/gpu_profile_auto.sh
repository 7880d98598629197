# ncu of the library's auto launch policy over NVLink (the bench default at N>=2):
# C2 (128 KiB spans) and C4 (8 KiB spans), GPU0 -> GPU1, one process.
M=nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvlrx__bytes_data_protocol.sum,nvlrx__bytes_packet_response_data_user.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes_packet_request_data_protocol.sum
for C in c2 c4; do
  Q="python tools/sweep.py --src-dev 0 --dst-dev 1 --profile-once --variants auto --config $C"
  $Q > gpurun_out/pa_plain_$C.log 2>&1 && timeout 600 ncu --set full --metrics $M --clock-control none --import-source on -k regex:pull_kernel -s 1 -c 1 -o gpurun_out/pa_prof_$C $Q > gpurun_out/pa_ncu_$C.log 2>&1; echo PROF_$C $?
done
