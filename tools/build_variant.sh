#!/bin/bash
# Builds build_variants/libqswg_<name>.so from the current objects with extra
# nvcc defines for cuda/taylor.cu (kernel experiments; load with QSWG_LIB_PATH).
#   tools/build_variant.sh <name> -DQSWG_KRON_MIN_BLOCKS=3 ...
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2003_02450_b200/csrc"
make -s -j8 >/dev/null
mkdir -p ../../build_variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC "$@" \
  -c cuda/taylor.cu -o /tmp/taylor_$name.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o ../../build_variants/libqswg_$name.so build/host/*.o build/capi.o $(ls build/cuda/*.o | grep -v taylor) \
  /tmp/taylor_$name.o -ldl -lpthread
