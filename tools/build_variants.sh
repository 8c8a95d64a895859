#!/usr/bin/env bash
# Build libgnetmon.so variants with extra -D flags for A/B runs (tools/ab_multi.sh):
#   tools/build_variants.sh name1 "-DFOO=1" name2 "-DFOO=2" ...
set -e
cd "$(dirname "$0")/.."
PKG=paper_1108_1785_b200
SRCS="$PKG/csrc/capi.cu $PKG/csrc/kernels.cu $PKG/csrc/netflow.cu $PKG/csrc/hosts.cu $PKG/csrc/registry.cpp $PKG/csrc/comm.cpp"
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  mkdir -p $PKG/lib/$name
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      -cudart static -Iinclude -ldl $flags -shared -o $PKG/lib/$name/libgnetmon.so $SRCS 2> $PKG/lib/$name/ptxas.log &
done
wait
ls -la $PKG/lib/*/libgnetmon.so
