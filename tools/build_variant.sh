#!/bin/bash
# Build the product library with extra nvcc defines into build/var_<name>/
# for A/B timing:  tools/build_variant.sh k2s8 -DWLM_K2_OWN_SLOTS=8
#   WLM_LIB_PATH=build/var_k2s8/libwarplm_b200.so python bench.py ...
set -eu
name=$1; shift
out=build/var_$name
mkdir -p $out
C=paper_2603_19371_b200/csrc
objs=""
for f in kernels hot_kernels engine ops synth slab io field64 generic; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Iinclude "$@" \
       -c $C/$f.cu -o $out/$f.o &
  objs="$objs $out/$f.o"
done
wait
printf 'const char* wlm_source_hash(void) { return "variant-%s"; }\n' "$name" > $out/src_hash.c
gcc -O2 -fPIC -c $out/src_hash.c -o $out/src_hash.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libwarplm_b200.so $objs $out/src_hash.o
echo "built $out/libwarplm_b200.so"
