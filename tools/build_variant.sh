#!/bin/bash
# Build a diagnostics/experiment variant of the library with extra -D flags on ONE source file, the
# other objects taken from the in-tree build.  Usage: bash tools/build_variant.sh <name> <src.cu> -DFOO ...
# -> build_variants/lib_<name>.so (select it with FAGP_LIB_PATH=...).
set -e
name=$1; src=$2; shift 2
mkdir -p build_variants/$name
objs=""
for o in paper_2403_12797_b200/build/*.o; do
  b=$(basename $o .o)
  if [ "$b" = "$src" ]; then continue; fi
  objs="$objs $o"
done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC "$@" -I include \
  -c paper_2403_12797_b200/csrc/$src -o build_variants/$name/$src.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build_variants/lib_$name.so $objs build_variants/$name/$src.o -lcudart
echo build_variants/lib_$name.so
