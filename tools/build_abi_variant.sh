#!/bin/bash
# Build a store-kernel variant library: only hcub_abi.o is recompiled with
# extra defines, K1 objects come from the default build.
#   tools/build_abi_variant.sh <name> <nvcc -D flags...>  -> paper_2511_01573_b200/libhcub_<name>.so
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2511_01573_b200/csrc"
b=build_$name
mkdir -p $b
for o in build/k1_fn*.o; do cp $o $b/; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -Xptxas -v "$@" \
  -I$(python3 -c "import nvidia.nccl as n, os; print(os.path.join(list(n.__path__)[0], 'include'))") -c hcub_abi.cu -o $b/hcub_abi.o > $b/hcub_abi.ptxas.txt 2>&1 || (cat $b/hcub_abi.ptxas.txt; false)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libhcub_$name.so $b/*.o -lcudart -ldl
grep -A3 "k3_classify" $b/hcub_abi.ptxas.txt | grep -E "Used|spill" | head -2
rm -rf "$b"
