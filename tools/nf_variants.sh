#!/bin/bash
# Build libh2b.so variants of quadrature.cu with -D macros (tuning only):
# tools/nf_variants.sh name "-DFOO=1" [name2 "flags2" ...]  -> _lib/variants/<name>.so
set -e
cd "$(dirname "$0")/.."
OBJ=paper_2001_05523_b200/_lib/obj
OUT=paper_2001_05523_b200/_lib/variants
mkdir -p $OUT
NVCC=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  $NVCC -c ${QSRC:-paper_2001_05523_b200/csrc/quadrature.cu} -o $OUT/$name.q.o -O3 -std=c++17 -Xcompiler -fPIC -I include \
    $ARCH -lineinfo --expt-relaxed-constexpr -Xptxas -v $flags 2>&1 | grep -A2 "k_blocks_slpILi9" | grep -E "spill|Used" | tr '\n' ' '; echo
  $NVCC -shared -o $OUT/$name.so $(ls $OBJ/*.o | grep -v quadrature.cu.o) $OUT/$name.q.o $ARCH \
    -lcudart_static -lrt -ldl -lpthread
  echo "built $OUT/$name.so ($flags)"
done
