# round 2, first GPU pass: build, smoke, the whole GPU suite (2 GPUs), a
# short N=1 and N=2 bench, and the early-loads A/B on back-to-back pulls.
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r02a_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02a_smoke.log 2>&1; echo SMOKE $?
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rs > gpurun_out/r02a_tests.log 2>&1; echo TESTS $?
tail -40 gpurun_out/r02a_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02a_b1.log 2>&1; echo B1 $?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 2 --steps 20 --warmup 5 --no-nccl > gpurun_out/r02a_b2.log 2>&1; echo B2 $?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 2 --steps 20 --warmup 5 --no-nccl --config c4 > gpurun_out/r02a_b2c4.log 2>&1; echo B2C4 $?
for e in 1 0; do
  timeout 600 python tools/small_requests.py --ipc --config c4 --tokens 128,1024,8192 --requests 16 --modes single,batch,merged --timing 0 --early $e >> gpurun_out/r02a_small.jsonl 2>> gpurun_out/r02a_small.err; echo SMALL$e $?
done
for f in r02a_b1 r02a_b2 r02a_b2c4; do grep '^{' gpurun_out/$f.log | cut -c1-400; done
cat gpurun_out/r02a_small.jsonl | cut -c1-600
