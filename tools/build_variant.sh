#!/bin/bash
# Build an alternate libdbf_b200.so with extra nvcc flags into tools/_x/<name>.so (debug/experiment
# variants; load with DBF_B200_LIB=tools/_x/<name>.so).  Usage: tools/build_variant.sh name -DFOO ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=tools/_x/$name; mkdir -p $out
for f in paper_2505_11076_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
       -I include -I paper_2505_11076_b200/csrc "$@" -c $f -o $out/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/_x/$name.so $out/*.o
echo tools/_x/$name.so
