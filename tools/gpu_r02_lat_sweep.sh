# 2-GPU box: C1 launch-shape sweep for the latency path (tools/native/kvd_latency,
# KVD_LAT_OPTS = extra kvd_peer_set calls), GPU0 -> GPU1, with in-kernel spans;
# plus the calibration tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_gpu_policy.py -rs > gpurun_out/r02l_tests.log 2>&1; echo TESTS $?; tail -3 gpurun_out/r02l_tests.log
nvcc -O2 -I include tools/native/kvd_latency.cu -L paper_2501_14743_b200 -lkvd \
  -Xlinker -rpath=$PWD/paper_2501_14743_b200 -o tools/native/kvd_latency 2>/dev/null
export KVD_LAT_C1_ONLY=1
OUT=gpurun_out/r02_lat_sweep.jsonl; : > $OUT
for o in "" "4=64" "4=128" "4=256" "4=512" "1=1024" "1=1024,4=64" "1=4096" "1=4096,4=64"; do
  KVD_LAT_OPTS="$o" timeout 120 tools/native/kvd_latency 0 1 2000 1 >> $OUT 2>&1
  KVD_LAT_OPTS="$o" timeout 120 tools/native/kvd_latency 0 1 2000 0 >> $OUT 2>&1
done
for e in 2 4 8; do timeout 120 tools/native/kvd_latency 0 1 2000 1 $e >> $OUT 2>&1; timeout 120 tools/native/kvd_latency 0 1 2000 0 $e >> $OUT 2>&1; done
cat $OUT
