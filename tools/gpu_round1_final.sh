python bench.py --steps 50 --warmup 5 > gpurun_out/f_n1.log 2>&1; echo N1 $?
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/f_n1b.log 2>&1; echo N1b $?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 2 --steps 50 --warmup 5 > gpurun_out/f_n2.log 2>&1; echo N2 $?
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/f_ref.log 2>&1; echo REF $?
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/f_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches_n1.csv $B > gpurun_out/f_ncu1.log 2>&1; echo LAUNCH $?
$B > gpurun_out/f_plain2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:pull_kernel -s 3 -c 1 -o gpurun_out/f_prof_n1 $B > gpurun_out/f_ncu2.log 2>&1; echo PROF $?
for f in f_n1 f_n1b f_n2 f_ref; do grep '^{' gpurun_out/$f.log | cut -c1-300; done
