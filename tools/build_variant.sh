#!/bin/bash
# Build libkvd.so with extra nvcc flags into paper_2501_14743_b200/ab/<name>/ (git-ignored;
# travels to the GPU box).  Load it with KVD_LIB_PATH=$PWD/paper_2501_14743_b200/ab/<name>/libkvd.so
#   tools/build_variant.sh <name> [nvcc flags...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
OUT=paper_2501_14743_b200/ab/$name
mkdir -p $OUT
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-fvisibility=hidden -cudart static -I include"
$NV "$@" -x cu -c paper_2501_14743_b200/csrc/kvd_core.cpp -o $OUT/core.o
$NV "$@" -x cu -c paper_2501_14743_b200/csrc/kvd_vmm.cpp -o $OUT/vmm.o
$NV "$@" -c paper_2501_14743_b200/csrc/kvd_pull.cu -o $OUT/pull.o
$NV -shared -cudart static -o $OUT/libkvd.so $OUT/core.o $OUT/vmm.o $OUT/pull.o \
    -Xlinker --version-script=paper_2501_14743_b200/csrc/kvd.map
rm $OUT/*.o
echo built $OUT/libkvd.so
