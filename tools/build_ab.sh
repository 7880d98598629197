#!/bin/bash
# Build A/B variants of libkvd.so with different load/store cache qualifiers
# into paper_2501_14743_b200/ab/<name>/libkvd.so (git-ignored; travels to the box).
set -e
cd "$(dirname "$0")/.."
OUT=paper_2501_14743_b200/ab
mkdir -p $OUT
build() {
  name=$1; shift
  mkdir -p $OUT/$name
  NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-fvisibility=hidden -cudart static -I include"
  $NV "$@" -x cu -c paper_2501_14743_b200/csrc/kvd_core.cpp -o $OUT/$name/core.o
  $NV "$@" -c paper_2501_14743_b200/csrc/kvd_pull.cu -o $OUT/$name/pull.o
  $NV -shared -cudart static -o $OUT/$name/libkvd.so $OUT/$name/core.o $OUT/$name/pull.o \
      -Xlinker --version-script=paper_2501_14743_b200/csrc/kvd.map
  rm $OUT/$name/*.o
  echo built $name
}
build base
build st_cs '-DKVD_ST_Q="st.global.cs"'
build ld_cs '-DKVD_LD_Q="ld.global.cs"' '-DKVD_ST_Q="st.global.cs"'
build ld_l2_256 '-DKVD_LD_Q="ld.global.nc.L1::no_allocate.L2::256B"'
build ld_lu '-DKVD_LD_Q="ld.global.lu"' '-DKVD_ST_Q="st.global.cs"'
