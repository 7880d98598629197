#!/bin/bash
# Build an A/B libkvd.so from the product sources with a patch applied (the
# product sources carry no experiment switches).  Output:
# paper_2501_14743_b200/ab/<name>/libkvd.so (git-ignored; travels to the GPU
# box).  Load it with KVD_LIB_PATH=$PWD/paper_2501_14743_b200/ab/<name>/libkvd.so
#   tools/build_patched.sh <name> tools/ab_patches/<file>.patch [more patches]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
TMP=$(mktemp -d)
mkdir -p $TMP/p
cp -r paper_2501_14743_b200/csrc $TMP/p/
cp -r include $TMP/
ROOT=$PWD
for p in "$@"; do (cd $TMP/p && patch -p1 -s < "$ROOT/$p"); done
OUT=paper_2501_14743_b200/ab/$name
mkdir -p $OUT
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-fvisibility=hidden -cudart static -I $TMP/include"
$NV -x cu -c $TMP/p/csrc/kvd_core.cpp -o $OUT/core.o
$NV -x cu -c $TMP/p/csrc/kvd_vmm.cpp -o $OUT/vmm.o
$NV -c $TMP/p/csrc/kvd_pull.cu -o $OUT/pull.o
$NV -shared -cudart static -o $OUT/libkvd.so $OUT/core.o $OUT/vmm.o $OUT/pull.o \
    -Xlinker --version-script=$TMP/p/csrc/kvd.map
rm -f $OUT/*.o
rm -rf $TMP
echo built $OUT/libkvd.so
