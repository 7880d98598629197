# A/B: early-read depth for long requests (C4 671 MB, C2 4 GiB) through bench.py
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
OUT=gpurun_out/r02_early_long.jsonl; : > $OUT
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=29700
for rep in 1 2; do
  for e in 2 4 6; do
    for c in c4 c2; do
      port=$((port+1)); st=100; [ $c = c2 ] && st=20
      v=$($T --master-port $port bench.py --gpus 2 --steps $st --warmup 5 --no-nccl --config $c --early $e 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'])")
      echo "{\"early\": $e, \"rep\": $rep, \"config\": \"$c\", \"value\": $v}" >> $OUT
    done
  done
done
cat $OUT
