# 2-GPU box: engine breakdown (entry seen -> handed over -> landed) by cluster size,
# then the engine tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvcc -O2 -I include tools/native/kvd_latency.cu -L paper_2501_14743_b200 -lkvd \
  -Xlinker -rpath=$PWD/paper_2501_14743_b200 -o tools/native/kvd_latency 2>/dev/null
export KVD_LAT_C1_ONLY=1
OUT=gpurun_out/r02_engine_sweep.jsonl; : > $OUT
for e in 4 8 12 16; do timeout 120 tools/native/kvd_latency 0 1 2000 1 $e >> $OUT 2>&1; timeout 120 tools/native/kvd_latency 0 1 2000 0 $e >> $OUT 2>&1; done
timeout 120 tools/native/kvd_latency 0 0 2000 1 8 >> $OUT 2>&1
timeout 120 tools/native/kvd_latency 0 0 2000 1 16 >> $OUT 2>&1
cat $OUT
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_gpu_engine.py -rs > gpurun_out/r02e_tests.log 2>&1; echo TESTS $?; tail -3 gpurun_out/r02e_tests.log
