#!/bin/bash
# Debug builds of libchemora (launch_fused prints + syncs): scripts/libchemora_dbg<suffix>.so
# usage: build_dbg.sh [suffix] [extra nvcc defines...]
set -e
R=/root/repo; C=$R/paper_1410_1764_b200/csrc; O=$R/paper_1410_1764_b200/build_obj
SUF=$1; shift || true
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I $R/include -I $C -DCHEMORA_DEBUG_FUSED "$@" -c $C/bssn_fused.cu -o /tmp/bssn_fused_dbg$SUF.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/scripts/libchemora_dbg$SUF.so $O/wave_stage.cu.o $O/wave_tma.cu.o \
  $O/wave_fused3.cu.o $O/bssn_stage.cu.o /tmp/bssn_fused_dbg$SUF.o $O/ghost_init_norms.cu.o $O/capi.cpp.o
