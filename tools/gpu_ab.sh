for v in base st_cs ld_cs ld_l2_256 ld_lu; do
  for dev in 0 1; do
    KVD_LIB_PATH=paper_2501_14743_b200/ab/$v/libkvd.so timeout 200 python tools/sweep.py --src-dev 0 --dst-dev $dev --tables fragmented --variants lsu --tiles 16384,65536 --threads 512 --iters 20 2>/dev/null | sed "s/^/$v dst$dev /" | cut -c1-40,150-260
  done
done
