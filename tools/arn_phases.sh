#!/bin/bash
# Phase timing of the fused Arnoldi step (profiling build, dev aid):
#   bash tools/arn_phases.sh [case]
# builds libpt_b200_prof.so with -DPT_ARN_PROFILE (globaltimer marks, device
# printf from block 0 and the last block) and runs one host-driven solve.
set -e
cd "$(dirname "$0")/../paper_1410_5910_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
  -I../../include --expt-relaxed-constexpr -DPT_ARN_PROFILE -shared \
  -o ../libpt_b200_prof.so pt_api.cu pt_exec.cu pt_gmres.cu pt_batch.cu pt_local.cu pt_plan.cpp
cd ../..
PT_GRAPH=0 PT_B200_LIB=paper_1410_5910_b200/libpt_b200_prof.so python tools/one_solve.py "${1:-c3}"
