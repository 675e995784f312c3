#!/bin/bash
# Build a variant of the engine library with extra nvcc defines:
#   tools/build_variant.sh tools/bin/out.so -DFO_POLY_OF_8=3 ...
out=$1; shift
cd "$(dirname "$0")/.." || exit 1
S=paper_2509_25401_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -shared "$@" -o "$out" \
  $S/fo_symbols.cu $S/fo_attention.cu $S/fo_attention_cs.cu $S/fo_gemm.cu $S/fo_elementwise.cu \
  $S/fo_policy.cu $S/fo_capi.cu
