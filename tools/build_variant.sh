#!/bin/bash
# Build an alternative library with extra nvcc defines into varlib/<name>.so (timing experiments only).
# usage: tools/build_variant.sh <name> "<extra nvcc flags>"
set -e
cd "$(dirname "$0")/.."
name=$1; shift
tmp=$(mktemp -d)
for f in paper_2311_17500_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $1 -c $f -o $tmp/$(basename $f .cu).o &
  pids="$pids $!"
done
for p in $pids; do wait $p || { echo "compile failed"; exit 1; }; done
mkdir -p varlib; nvcc -shared -gencode arch=compute_100a,code=sm_100a -o varlib/$name.so $tmp/*.o -lcudart
rm -rf $tmp
echo built varlib/$name.so
