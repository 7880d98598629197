# f1 batched drain over NVLink (C3, one pair): mover / ring shapes, one bench
# line per configuration.  Configurations come one per line on stdin, e.g.
#   printf -- '--variant tma --threads 64 --stages 3 --tile 32768 --max-ctas 64\n' | bash tools/batch_sweep.sh
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
i=0
while IFS= read -r args; do
  [ -z "$args" ] && continue
  i=$((i+1))
  $T --master-port $((29810+i)) bench.py --gpus 2 --config c3 --batch --steps 5 --warmup 3 \
     --no-nccl --no-cpu-baseline $args > gpurun_out/bs_$i.log 2>&1 < /dev/null
  grep "^{" gpurun_out/bs_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'args': '$args', 'value': d['value'], 'kernel': d['roofline']['achieved'], 'variant': d['config']['variant'], 'ctas': d['config']['ctas'], 'threads': d['config']['threads'], 'parity': d['parity']}))"
done
