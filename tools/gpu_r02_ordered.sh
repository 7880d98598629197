# KVD_OPT_ENGINE_ORDERED: the engine tests (incl. stream order), and C1
# host-to-host latency with the ordered engine vs unordered vs launched.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_gpu_engine.py -x > gpurun_out/r02_ordered_tests.log 2>&1; echo T $?; tail -15 gpurun_out/r02_ordered_tests.log
nvcc -O2 -I include tools/native/kvd_latency.cu -L paper_2501_14743_b200 -lkvd \
  -Xlinker -rpath=$PWD/paper_2501_14743_b200 -o tools/native/kvd_latency 2>/dev/null
export KVD_LAT_C1_ONLY=1
OUT=gpurun_out/r02_ordered_latency.jsonl; : > $OUT
for rep in 1 2; do
  for d in 1 0; do
    timeout 120 tools/native/kvd_latency 0 $d 2000 0 >> $OUT 2>&1
    timeout 120 tools/native/kvd_latency 0 $d 2000 0 16 >> $OUT 2>&1
    KVD_LAT_OPTS="11=1" timeout 120 tools/native/kvd_latency 0 $d 2000 0 16 >> $OUT 2>&1
  done
done
cut -c1-330 $OUT
