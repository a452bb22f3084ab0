#!/bin/bash
# Experimental builds of the library with compile-time knobs (profiling only).
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/_variants
for spec in "$@"; do
  name=${spec%%=*}; flags=${spec#*=}
  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 --expt-relaxed-constexpr \
       -shared -Xcompiler -fPIC $flags -o tools/_variants/lib_$name.so paper_2111_09947_b200/csrc/maskmul_abi.cu &
done
wait
