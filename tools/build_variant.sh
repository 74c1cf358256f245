#!/bin/bash
# A/B experiments: build the library with extra -D flags into
# paper_1701_05975_b200/lib_var/libwbc_<name>.so (select it with WBC_LIB=...).
#   tools/build_variant.sh <name> "-DWBC_FLAT_RELAX_U=1 ..."
set -e
name=$1; shift
defs="$*"
cd "$(dirname "$0")/../paper_1701_05975_b200"
make -s lib/libwbc_b200.so
mkdir -p build_var/$name lib_var
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC \
  -I../include -Icsrc --expt-relaxed-constexpr $defs -c csrc/wbc_gpu.cu -o build_var/$name/wbc_gpu.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o lib_var/libwbc_$name.so \
  build_var/$name/wbc_gpu.o build/host_graph.o build/host_generate.o build/host_capi.o build/host_engine.o \
  build/host_report.o -lcudart_static -lrt -ldl -lpthread
echo lib_var/libwbc_$name.so
