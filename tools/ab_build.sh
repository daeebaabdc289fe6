#!/bin/bash
# Build the committed (HEAD) sources as paper_2305_09493_b200/libskgpu_base.so
# for same-box A/B timing against the working tree's libskgpu.so
# (SKGPU_LIB=paper_2305_09493_b200/libskgpu_base.so selects it).
set -e
cd "$(dirname "$0")/.."
tmp=$(mktemp -d)
git archive HEAD paper_2305_09493_b200/csrc include | tar -x -C "$tmp"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -diag-suppress 20091 -o paper_2305_09493_b200/libskgpu_base.so "$tmp/paper_2305_09493_b200/csrc/skg_api.cu"
rm -rf "$tmp"
