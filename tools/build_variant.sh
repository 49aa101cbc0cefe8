#!/bin/bash
# Builds a variant of libssjoin.so with extra nvcc -D flags for A/B timing:
#   tools/build_variant.sh NAME "-DSSJB_SUSPEND_NS=0 ..."
# -> paper_1711_07295_b200/lib/variants/libssjoin_NAME.so (use with SSJB_LIB=...)
set -e
NAME=$1; shift
DEFS="$*"
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_1711_07295_b200/csrc
B=$ROOT/paper_1711_07295_b200/build/variant_$NAME
mkdir -p $B $ROOT/paper_1711_07295_b200/lib/variants
make -s -C $C -j8 >/dev/null
NVCC=${CUDA_HOME:-/usr/local/cuda}/bin/nvcc
$NVCC -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -ccbin g++ -Xcompiler -fPIC,-fvisibility=hidden \
  --expt-relaxed-constexpr $DEFS -c $C/engine.cu -o $B/engine.o
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -ccbin g++ -cudart static -Xlinker --version-script=$C/exports.map \
  -Xlinker -Bsymbolic -o $ROOT/paper_1711_07295_b200/lib/variants/libssjoin_$NAME.so \
  $ROOT/paper_1711_07295_b200/build/host_core.o $ROOT/paper_1711_07295_b200/build/capi.o $B/engine.o -lpthread -ldl -lrt
echo built lib/variants/libssjoin_$NAME.so
