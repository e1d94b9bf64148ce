#!/bin/bash
# Build A/B variants of the library: tools/ab_build.sh name "-DFOO=1" [name2 "-DBAR=2" ...]
# Outputs build/ab/<name>.so (git-ignored; travels to the GPU box with gpurun).
set -e
cd "$(dirname "$0")/.."
mkdir -p build/ab
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
    -Iinclude $flags -o build/ab/$name.so paper_1905_09071_b200/csrc/ttagg_b200.cu 2>&1 | grep -v -i "warning\|prefetch_l2\|^ *\^\|^$\|Remark" || true &
done
wait
ls -la build/ab/
