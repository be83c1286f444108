#!/bin/bash
# Build a variant of the sweep library into variants/NAME.so with extra nvcc
# flags (e.g. -DKVSIM_COOP_CHAIN=1) for in-process A/B (tools/ab_inproc.py).
NAME=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++20 \
  -Xcompiler -fPIC,-ffp-contract=off -I$R/include -shared "$@" -o $R/variants/$NAME.so \
  $R/paper_2411_05555_b200/csrc/kvsim_sweep.cu $R/paper_2411_05555_b200/csrc/kvsim_sweep_full.cu \
  $R/paper_2411_05555_b200/csrc/perfmodel.cpp
