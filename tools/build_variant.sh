#!/bin/bash
# Dev helper: build a variant of libkvgpu.so with extra nvcc defines into
# var_libs/ (gitignored; travels to the GPU box). Usage:
#   tools/build_variant.sh prof -DKVG_PROFILE
set -e
cd "$(dirname "$0")/.."
name=$1; shift
python -m paper_2601_22705_b200.build >/dev/null
mkdir -p var_libs
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false -prec-div=true -Xcompiler -fPIC,-fvisibility=hidden"
nvcc $F "$@" -c paper_2601_22705_b200/csrc/engine.cu -o var_libs/engine_$name.o
nvcc $F "$@" -c paper_2601_22705_b200/csrc/capi.cu -o var_libs/capi_$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o var_libs/libkvgpu_$name.so \
  var_libs/engine_$name.o var_libs/capi_$name.o build/controllers.o build/host.o build/artifacts.o
echo var_libs/libkvgpu_$name.so
