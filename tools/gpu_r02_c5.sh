# C5 sweep with the final kernel at one pair (best NCCL variant per point),
# and the interference of the default pull with a concurrent decode GEMM.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29701 tools/c5_sweep.py --iters 10 > gpurun_out/r02_c5_sweep_n2.jsonl 2> gpurun_out/r02_c5_err.log; echo C5 $?
timeout 900 python tools/interference.py > gpurun_out/r02_interference.jsonl 2> gpurun_out/r02_interf_err.log; echo INTERF $?
python -c "
import json
for l in open('gpurun_out/r02_c5_sweep_n2.jsonl'):
    if not l.startswith('{'): continue
    d=json.loads(l); print(d['model'], d['block_size'], d['run_blocks'], d['pull_gbs_per_pair'], d['pull_nocoalesce_gbs_per_pair'], d.get('nccl_best_transfer'), d.get('pull_vs_best_nccl'), d.get('pull_vs_nccl_n0_ceiling'), d['parity'], d.get('nccl_parity'))
"
tail -3 gpurun_out/r02_interference.jsonl
tail -3 gpurun_out/r02_c5_err.log
