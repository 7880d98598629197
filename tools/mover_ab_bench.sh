T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
i=0
while IFS= read -r args; do
  i=$((i+1))
  $T --master-port $((29850+i)) bench.py --gpus 2 --steps 10 --warmup 3 --no-nccl --no-cpu-baseline $args > gpurun_out/m_$i.log 2>&1 < /dev/null
  grep "^{" gpurun_out/m_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'args': '$args', 'value': d['value'], 'kernel': d['roofline']['achieved'], 'variant': d['config']['variant'], 'ctas': d['config']['ctas'], 'threads': d['config']['threads']}))"
done <<'CFG'
--config c2
--config c2 --variant lsu32
--config c3 --batch
--config c3 --batch --variant lsu32
--config c3
--config c3 --variant lsu32
CFG
