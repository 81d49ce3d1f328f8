#!/bin/bash
# tools/build_variant.sh NAME "-DFLAG=V ..."  ->  tools/variant/NAME/libsmoe_b200.so
# (kernels.cu rebuilt with extra defines, linked with the package's other objects;
# tools only — loaded by tools/kbench.py through SMOE_LIB)
set -e
cd "$(dirname "$0")/../paper_2603_19289_b200/csrc"
make -j4 >/dev/null
out=../../tools/variant/$1
mkdir -p "$out"
ARCH="-gencode arch=compute_100a,code=sm_100a"
/usr/local/cuda/bin/nvcc $ARCH -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC $2 -c kernels.cu -o "$out/kernels.o"
/usr/local/cuda/bin/nvcc $ARCH -shared -o "$out/libsmoe_b200.so" "$out/kernels.o" build/prefill.o build/prefill_tc.o \
  build/engine.o build/capi.o build/report.o build/xpack.o build/train_dev.o build/train.o -L/usr/local/cuda/lib64 -lcudart_static -lpthread -lrt -ldl
echo "built $out"
