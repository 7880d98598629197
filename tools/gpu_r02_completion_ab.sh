# A/B (timing only, unsound): C1 launched latency without the completion chain
# (tools/ab_patches/no_completion_chain.patch) vs the product, GPU0 -> GPU1 and loopback
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/build_patched.sh nochain tools/ab_patches/no_completion_chain.patch > /dev/null
export KVD_LAT_C1_ONLY=1
OUT=gpurun_out/r02_completion_ab.jsonl; : > $OUT
for lib in base nochain; do
  if [ $lib = base ]; then D=$PWD/paper_2501_14743_b200; else D=$PWD/paper_2501_14743_b200/ab/$lib; fi
  nvcc -O2 -I include tools/native/kvd_latency.cu -L $D -lkvd -Xlinker -rpath=$D -o /tmp/lat_$lib 2>/dev/null
  for rep in 1 2; do
    echo "{\"lib\": \"$lib\"}" >> $OUT
    timeout 120 /tmp/lat_$lib 0 1 2000 0 >> $OUT 2>&1
    timeout 120 /tmp/lat_$lib 0 0 2000 0 >> $OUT 2>&1
  done
done
cut -c1-200 $OUT
