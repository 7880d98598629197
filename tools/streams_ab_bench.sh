# KVD_OPT_STREAMS A/B through bench.py over one NVLink pair (and C4 over 2 pairs)
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
while IFS= read -r line; do
  i=$((i+1)); n=${line%% *}; args=${line#* }
  $T --nproc-per-node $n --master-port $((29900+i)) bench.py --gpus $n --steps 20 --warmup 3 --no-nccl --no-cpu-baseline $args > gpurun_out/sab_$i.log 2>&1 < /dev/null
  grep "^{" gpurun_out/sab_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'n': $n, 'args': '$args', 'value': d['value'], 'gbs_per_pair': d['gbs_per_pair'], 'kernel': d['roofline']['achieved'], 'e2e': d['e2e']['value'], 'p50_ms': d['p50_latency_ms'], 'parity': d['parity']}))"
done <<'CFG'
2 --config c2
2 --config c2 --streams 2
2 --config c4
2 --config c4 --streams 2
2 --config c3
2 --config c3 --streams 2
2 --config c3 --batch
CFG
