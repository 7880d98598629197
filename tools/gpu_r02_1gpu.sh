# what the driver runs at round end, on a one-GPU box: the GPU suite, smoke, bench N=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02p_smoke.log 2>&1; echo SMOKE $?
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rs --durations=15 > gpurun_out/r02p_tests.log 2>&1; echo TESTS $?
tail -30 gpurun_out/r02p_tests.log
timeout 900 python bench.py > gpurun_out/r02p_bench.log 2>&1; echo BENCH $?
grep '^{' gpurun_out/r02p_bench.log | cut -c1-400
