#!/bin/bash
# A/B build of libmtnn_b200.so with extra nvcc -D flags (for gemm_tc.cu, or the
# .cu files listed in $FILES):
#   [FILES="gemm_tc.cu fixup.cu"] tools/build_variant.sh NAME -DFOO=1 ...
#   ->  build/variants/NAME/libmtnn_b200.so
# (select it with MTNN_B200_LIB=... ; the in-tree library is untouched)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
python paper_1702_03192_b200/build.py > /dev/null
out=build/variants/$name; mkdir -p $out
files=${FILES:-gemm_tc.cu}
objs=$(ls build/mtnn_b200/*.o)
for f in $files; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Xcompiler -ffp-contract=off --expt-relaxed-constexpr -Iinclude "$@" \
    -c paper_1702_03192_b200/csrc/$f -o $out/$f.o
  objs=$(echo "$objs" | grep -v "/$f.o")
  objs="$objs $out/$f.o"
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libmtnn_b200.so $objs -lpthread -ldl -lrt
echo $out/libmtnn_b200.so
