#!/bin/bash
# dev: build the library from the current tree into build/<name>/ (A/B variants)
cd "$(dirname "$0")/.."
mkdir -p build/$1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -cudart static -Iinclude ${@:2} -o build/$1/libtriadcensus.so paper_1603_02655_b200/csrc/*.cu -ldl
