#!/bin/bash
# Build a variant of the library for A/B runs: tools/build_variant.sh NAME [SRC_DIR] [nvcc flags...]
# -> tools/variants/lib_NAME.so (select it with CTW_B200_LIB=...).
set -e
name=$1; shift
dir=${1:-paper_2311_04996_b200/csrc}; shift || true
mkdir -p tools/variants
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared \
  -I paper_2311_04996_b200/csrc -o tools/variants/lib_$name.so "$@" \
  $dir/ctw_api.cu $dir/ctw_kernels.cu $dir/ctw_kernels_wide.cu $dir/ctw_kernels_wide64.cu $dir/ctw_lattice.cu $dir/ctw_history.cu paper_2311_04996_b200/csrc/ctw_graphbuild.cpp
