#!/bin/bash
# Build a K1 variant library for measurement: only the K1 object of integrand
# kind $FN (default 2 = f2) is
# recompiled with extra defines, the rest is taken from the default build.
#   tools/build_k1_variant.sh <name> '<nvcc -D flags>'   -> paper_2511_01573_b200/libhcub_<name>.so
set -e
name=$1; shift
extra=("$@")
cd "$(dirname "$0")/../paper_2511_01573_b200/csrc"
b=build_$name
mkdir -p $b
FN=${FN:-2}
for o in build/*.o; do [[ $(basename $o) == k1_fn$FN.o ]] || cp $o $b/; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -Xptxas -v "${extra[@]}" \
  -DHCUB_FN=$FN -c k1_inst.cu -o $b/k1_fn$FN.o > $b/k1_fn$FN.ptxas.txt 2>&1 || (cat $b/k1_fn$FN.ptxas.txt; false)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libhcub_$name.so $b/*.o -lcudart -ldl
cp $b/k1_fn$FN.ptxas.txt ../libhcub_$name.ptxas.txt
grep -A2 "${GREPK:-k1_gm_evalILi5ELi2\|k1_gm_evalILi8ELi2}" $b/k1_fn$FN.ptxas.txt | grep -E "Used|spill" | head -4
rm -rf "$b"  # objects are not needed on the GPU box (snapshot size)
