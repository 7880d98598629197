# round 2 closing evidence on a 4-GPU box with the final kernel (guided
# claims): N = 2 (GPUs 0,1) and N = 4 bench lines for C2 / C4 / C3 / C3
# batched / C1, each with the NCCL baselines and the link calibration.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T="timeout 1200 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
p=29500
run() { n=$1; shift; tag=$1; shift; p=$((p+1))
  if [ $n = 2 ]; then CUDA_VISIBLE_DEVICES=0,1 $T --nproc-per-node 2 --master-port $p bench.py --gpus 2 "$@" > gpurun_out/r02f_n${n}_$tag.log 2>&1
  else $T --nproc-per-node 4 --master-port $p bench.py --gpus 4 "$@" > gpurun_out/r02f_n${n}_$tag.log 2>&1; fi
  echo "N$n $tag $?"; }
for n in 2 4; do
  run $n c2 --steps 20 --warmup 5
  run $n c4 --steps 100 --warmup 5 --config c4
  run $n c3 --steps 5 --warmup 3 --config c3
  run $n c3b --steps 5 --warmup 3 --config c3 --batch --no-nccl
  run $n c1 --steps 100 --warmup 5 --config c1 --engine 16
done
for f in gpurun_out/r02f_*.log; do echo $f; grep '^{' $f | cut -c60-160; done
