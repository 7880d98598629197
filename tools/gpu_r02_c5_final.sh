# C5 sweep with the final kernel (guided claims) at 1 and 2 pairs, one 4-GPU box.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29751 tools/c5_sweep.py --iters 10 > gpurun_out/r02_c5_final_n2.jsonl 2> gpurun_out/r02_c5f_err2.log; echo C5N2 $?
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29752 tools/c5_sweep.py --iters 10 > gpurun_out/r02_c5_final_n4.jsonl 2> gpurun_out/r02_c5f_err4.log; echo C5N4 $?
for n in 2 4; do python - <<PY
import json
rows=[json.loads(l) for l in open("gpurun_out/r02_c5_final_n$n.jsonl") if l.startswith("{")]
for m in ("7b","70b"):
    xs=[r for r in rows if r["model"]==m]
    print($n, m, len(xs), min(r["pull_gbs_per_pair"] for r in xs), max(r["pull_gbs_per_pair"] for r in xs), min(r.get("pull_vs_best_nccl",0) for r in xs), max(r.get("pull_vs_best_nccl",0) for r in xs), all(r["parity"] for r in xs))
PY
done
