#!/bin/bash
# Build a variant of the engine library with extra nvcc defines applied to ONE
# translation unit; the others are linked from the current build objects:
#   tools/build_variant.sh tools/bin/out.so fo_gemm.cu -DFO_GO_PF=2 ...
out=$1; tu=$2; shift 2
cd "$(dirname "$0")/.." || exit 1
python -m paper_2509_25401_b200.build >/dev/null || exit 1
S=paper_2509_25401_b200/csrc
B=paper_2509_25401_b200/build
mkdir -p "$(dirname "$out")"
tmpo=$(mktemp --suffix=.o)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -c "$@" -o "$tmpo" $S/$tu || exit 1
objs=""
stem=${tu%.cu}
for o in $(python -c "
import paper_2509_25401_b200.build as b
print(' '.join(str(b._obj(s)) for s in b.SOURCES if not s.startswith('$stem.')))"); do objs="$objs $o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" $tmpo $objs
rm -f "$tmpo"
