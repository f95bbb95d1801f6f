#!/bin/bash
# Build libh2b.so variants of matvec.cu with different -D macros into
# paper_2001_05523_b200/_lib/variants/<name>.so (tuning experiments only).
# usage: tools/mv_variants.sh name "-DFOO=1 -DBAR=2" [name2 "flags2" ...]
set -e
cd "$(dirname "$0")/.."
OBJ=paper_2001_05523_b200/_lib/obj
OUT=paper_2001_05523_b200/_lib/variants
mkdir -p $OUT
NVCC=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  $NVCC -c ${SRC:-paper_2001_05523_b200/csrc/matvec.cu} -o $OUT/$name.o -O3 -std=c++17 -Xcompiler -fPIC -I include \
    $ARCH -lineinfo --expt-relaxed-constexpr $flags
  $NVCC -shared -o $OUT/$name.so $(ls $OBJ/*.o | grep -v matvec.cu.o) $OUT/$name.o $ARCH \
    -lcudart_static -lrt -ldl -lpthread
  echo "built $OUT/$name.so ($flags)"
done
