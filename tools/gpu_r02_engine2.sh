# 2-GPU box: engine with shared-memory layer bases (C1 latency, engine tests),
# then the back-to-back short-pull shape sweep.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvcc -O2 -I include tools/native/kvd_latency.cu -L paper_2501_14743_b200 -lkvd \
  -Xlinker -rpath=$PWD/paper_2501_14743_b200 -o tools/native/kvd_latency 2>/dev/null
export KVD_LAT_C1_ONLY=1
OUT=gpurun_out/r02_engine_smem_bases.jsonl; : > $OUT
for rep in 1 2; do for e in 8 16; do
  timeout 120 tools/native/kvd_latency 0 1 2000 0 $e >> $OUT 2>&1
  timeout 120 tools/native/kvd_latency 0 1 2000 1 $e >> $OUT 2>&1
done; done
timeout 120 tools/native/kvd_latency 0 0 2000 0 16 >> $OUT 2>&1
timeout 120 tools/native/kvd_latency 0 0 2000 1 16 >> $OUT 2>&1
cut -c1-260 $OUT
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_engine.py tests/test_gpu_multiprocess.py -k "engine" -rs > gpurun_out/r02e2_tests.log 2>&1; echo TESTS $?; tail -3 gpurun_out/r02e2_tests.log
unset KVD_LAT_C1_ONLY
bash tools/gpu_r02_short_sweep.sh
