mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_engine.py -x -rs -s > gpurun_out/r02h_engine_tests.log 2>&1; echo ENGINE_TESTS $?
tail -4 gpurun_out/r02h_engine_tests.log
for e in 4 8 16 32; do timeout 300 tools/native/kvd_latency 0 1 2000 0 $e >> gpurun_out/r02h_lat.jsonl 2>&1; done
for e in 8 16; do timeout 300 tools/native/kvd_latency 0 1 2000 1 $e >> gpurun_out/r02h_lat.jsonl 2>&1; done
timeout 300 tools/native/kvd_latency 0 1 2000 1 0 >> gpurun_out/r02h_lat.jsonl 2>&1
for e in 8; do timeout 300 tools/native/kvd_latency 0 0 2000 0 $e >> gpurun_out/r02h_lat.jsonl 2>&1; done
cut -c1-360 gpurun_out/r02h_lat.jsonl
