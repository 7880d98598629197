# bench.py --pairing ring on 4 GPUs (and 2): N concurrent pulls through
# NVSwitch, every GPU's ingress and egress carrying one -- at N = 4 as many
# concurrent pulls as the 4P:4D rail pairing at N = 8.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T="timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
$T --nproc-per-node 4 --master-port 29611 bench.py --gpus 4 --steps 20 --warmup 5 --pairing ring > gpurun_out/r02_ring_n4_c2.log 2>&1; echo R4C2 $?
$T --nproc-per-node 4 --master-port 29612 bench.py --gpus 4 --steps 100 --warmup 5 --pairing ring --config c4 > gpurun_out/r02_ring_n4_c4.log 2>&1; echo R4C4 $?
$T --nproc-per-node 4 --master-port 29613 bench.py --gpus 4 --steps 5 --warmup 3 --pairing ring --config c3 > gpurun_out/r02_ring_n4_c3.log 2>&1; echo R4C3 $?
CUDA_VISIBLE_DEVICES=0,1 $T --nproc-per-node 2 --master-port 29614 bench.py --gpus 2 --steps 20 --warmup 5 --pairing ring > gpurun_out/r02_ring_n2_c2.log 2>&1; echo R2C2 $?
for f in r02_ring_n4_c2 r02_ring_n4_c4 r02_ring_n4_c3 r02_ring_n2_c2; do grep '^{' gpurun_out/$f.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$f', d['value'], d['gbs_per_pair'], r['per_pair_achieved'], r['frac'], r['peak'], d['parity'], d['clocks']['reasons'])"; tail -2 gpurun_out/$f.log | cut -c1-200; done
