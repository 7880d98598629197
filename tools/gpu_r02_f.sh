# round 2: the resident pull engine -- tests, C1 latency, and a regression
# pass over the suites touched by the host changes.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_engine.py -x -rs -s > gpurun_out/r02f_engine_tests.log 2>&1; echo ENGINE_TESTS $?
tail -15 gpurun_out/r02f_engine_tests.log
for e in 0 1 2 4 8 16; do timeout 300 tools/native/kvd_latency 0 1 2000 0 $e >> gpurun_out/r02f_lat.jsonl 2>&1; done
for e in 0 8; do timeout 300 tools/native/kvd_latency 0 0 2000 0 $e >> gpurun_out/r02f_lat.jsonl 2>&1; done
cat gpurun_out/r02f_lat.jsonl
timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_gpu_multiprocess.py tests/test_gpu_concurrency.py tests/test_gpu_release.py tests/test_gpu_parity.py -rs > gpurun_out/r02f_tests.log 2>&1; echo TESTS $?
tail -5 gpurun_out/r02f_tests.log
