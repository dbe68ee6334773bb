#!/bin/bash
# Build libcvx variants with extra -D flags into variants/ (git-ignored): tools/build_variants.sh NAME "FLAGS" ...
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
    -shared --cudart static $flags -I include -o variants/libcvx_$name.so paper_2410_21149_b200/csrc/*.cu &
done
wait
ls -la variants/
