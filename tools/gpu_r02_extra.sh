# round 2 final-kernel refresh of the secondary tables: many short requests
# (single pulls vs batched drain vs one merged request, prefill in a second
# process), f4 head-slice pulls, push (f2) with the auto policy, and the
# interference of the default pull with a concurrent decode GEMM.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/small_requests.py --ipc --config c4 --tokens 128,1024 --requests 16 > gpurun_out/r02x_small.jsonl 2>gpurun_out/r02x.err; echo SMALL4 $?
timeout 600 python tools/small_requests.py --ipc --config c2 --tokens 128,512,4096 --requests 16 >> gpurun_out/r02x_small.jsonl 2>>gpurun_out/r02x.err; echo SMALL2 $?
timeout 600 python tools/heads_probe.py > gpurun_out/r02x_heads.json 2>>gpurun_out/r02x.err; echo HEADS $?
timeout 600 python tools/sweep.py --mode push --variants auto --config c2 > gpurun_out/r02x_push.jsonl 2>>gpurun_out/r02x.err; echo PUSH $?
timeout 600 python tools/sweep.py --mode pull --variants auto --config c2 >> gpurun_out/r02x_push.jsonl 2>>gpurun_out/r02x.err; echo PULL $?
timeout 900 python tools/interference.py > gpurun_out/r02x_interference.jsonl 2>>gpurun_out/r02x.err; echo INTERF $?
cut -c1-300 gpurun_out/r02x_small.jsonl; cat gpurun_out/r02x_heads.json; cut -c1-300 gpurun_out/r02x_push.jsonl; cat gpurun_out/r02x_interference.jsonl; tail -5 gpurun_out/r02x.err
