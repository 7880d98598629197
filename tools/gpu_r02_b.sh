# round 2: timeline breakdown of back-to-back pulls (early loads on/off), C1
# latency through the C ABI, and the new bench (NCCL N0/N3, latency, calibration).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for e in 1 0; do
  timeout 600 python tools/timeline.py --config c4 --tokens 128,1024,8192 --requests 24 --early $e >> gpurun_out/r02b_timeline.jsonl 2>>gpurun_out/r02b_err.log; echo TL$e $?
  timeout 600 python tools/timeline.py --config c2 --tokens 128,1024 --requests 24 --early $e >> gpurun_out/r02b_timeline.jsonl 2>>gpurun_out/r02b_err.log; echo TLc2$e $?
done
timeout 300 tools/native/kvd_latency 0 1 2000 0 > gpurun_out/r02b_lat01.jsonl 2>&1; echo LAT $?
timeout 300 tools/native/kvd_latency 0 1 2000 1 > gpurun_out/r02b_lat01_t.jsonl 2>&1; echo LATT $?
timeout 300 tools/native/kvd_latency 0 0 2000 1 > gpurun_out/r02b_lat00_t.jsonl 2>&1; echo LAT0 $?
T="timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$T --master-port 29661 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02b_n2_c2.log 2>&1; echo N2C2 $?
$T --master-port 29662 bench.py --gpus 2 --steps 50 --warmup 5 --config c1 > gpurun_out/r02b_n2_c1.log 2>&1; echo N2C1 $?
$T --master-port 29663 bench.py --gpus 2 --steps 20 --warmup 5 --config c4 > gpurun_out/r02b_n2_c4.log 2>&1; echo N2C4 $?
cat gpurun_out/r02b_timeline.jsonl
cat gpurun_out/r02b_lat*.jsonl
for f in r02b_n2_c2 r02b_n2_c1 r02b_n2_c4; do grep '^{' gpurun_out/$f.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['config']['workload'][:3], d['value'], d['p50_latency_ms'], json.dumps(d.get('latency')), json.dumps(d['roofline'])[:600], json.dumps(d.get('calibration')), json.dumps(d.get('nccl_baseline')))
"; tail -3 gpurun_out/$f.log; done
tail -5 gpurun_out/r02b_err.log
