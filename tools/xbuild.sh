#!/bin/bash
# Build an experimental libtagg variant: tools/xbuild.sh <name> [-DFLAG ...] -> xlib/<name>.so
# (A/B timing with tools/quick.py xlib/a.so xlib/b.so; not part of the product.)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
mkdir -p "$ROOT/xlib"
C=$ROOT/paper_2508_16584_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I"$ROOT/include" -cudart static \
  "$@" -shared -o "$ROOT/xlib/$name.so" $C/tagg_gemm.cu $C/tagg_pad.cu $C/tagg_quant.cu $C/tagg_wgrad.cu $C/tagg_moe.cu $C/tagg_plan.cpp
