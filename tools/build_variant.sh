#!/bin/bash
# Build an A/B variant of libfmmbem_b200.so with extra defines for one source file:
#   tools/build_variant.sh NAME FILE.cu "-DFOO=1"   ->  build/variants/libfmmbem_NAME.so
# then run with FMMBEM_LIB=build/variants/libfmmbem_NAME.so
set -e
NAME=$1; SRC=$2; DEFS=$3
cd "$(dirname "$0")/../paper_1506_05957_b200/csrc"
OUT=../../build/variants; mkdir -p $OUT
OBJS=""
for f in ../../build/obj/*.o; do b=$(basename $f .o); if [ "$b.cu" != "$SRC" ]; then OBJS="$OBJS $f"; fi; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off,-O2 \
     --expt-relaxed-constexpr $DEFS -c $SRC -o $OUT/$NAME.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libfmmbem_$NAME.so $OUT/$NAME.o $OBJS -ldl
echo $OUT/libfmmbem_$NAME.so
