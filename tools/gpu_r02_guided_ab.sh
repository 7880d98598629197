# A/B: guided tile claims (single tiles for the last claims of a pull,
# tools/ab_patches/guided_claims.patch) vs the product: C4 / C2 through
# bench.py (100 steps) and the short-pull timeline, two reps, same box.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/build_patched.sh guided tools/ab_patches/guided_claims.patch > /dev/null
OUT=gpurun_out/r02_guided_ab.jsonl; : > $OUT
T="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=29300
for rep in 1 2; do
  for lib in base guided; do
    if [ $lib = base ]; then unset KVD_LIB_PATH; else export KVD_LIB_PATH=$PWD/paper_2501_14743_b200/ab/guided/libkvd.so; fi
    for c in c4 c2; do
      port=$((port+1))
      st=100; [ $c = c2 ] && st=20
      v=$($T --master-port $port bench.py --gpus 2 --steps $st --warmup 5 --no-nccl --config $c 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'])")
      echo "{\"lib\": \"$lib\", \"rep\": $rep, \"config\": \"$c\", \"value\": $v}" >> $OUT
    done
    timeout 300 python tools/timeline.py --config c4 --tokens 128,1024,8192 --requests 24 --early 2 --label $lib >> gpurun_out/r02_guided_tl.jsonl 2>/dev/null
  done
done
unset KVD_LIB_PATH
cat $OUT
python - <<'PY'
import json
for l in open("gpurun_out/r02_guided_tl.jsonl"):
    d = json.loads(l); m = d["us_median"]
    print(f'{d["label"]:7s} {d["tokens"]:5d} per={d["gbs_per_period"]:6.1f} span={m["span"]:7.2f} period={m["period"]:7.2f} handoff={m["handoff"]:5.2f}')
PY
