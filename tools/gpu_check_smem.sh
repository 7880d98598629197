set -x
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests9.log 2>&1; echo TESTS $?; tail -3 gpurun_out/gpu_tests9.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 tools/c5_sweep.py --iters 10 --models 70b --bs 8,16 --runs 1,2,4 --no-nccl > gpurun_out/c5_small.jsonl 2> gpurun_out/c5_small.err; echo C5 $?
cut -c1-250 gpurun_out/c5_small.jsonl
timeout 300 python tools/sweep.py --src-dev 0 --dst-dev 0 --tables fragmented --variants lsu,lsu32,tma --tiles 16384,32768,65536 --threads 32,256,512 --stages 3,6 --ctas 0,148,296 --iters 10 > gpurun_out/sweep_loop.log 2>&1; echo LOOP $?
sort -t: -k11 gpurun_out/sweep_loop.log | cut -c40-250 | tail -60
