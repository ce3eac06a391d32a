#!/bin/bash
# Profiling build (not product): libgoom with clock64 stamps in the fused one-SM LMME
# (GOOM_TC_TRACE) -> tools/bin/libgoom_trace.so, read by tools/tc_trace.py
set -e
cd "$(dirname "$0")/../paper_2510_03426_b200/csrc"
make -s
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -ftz=false -prec-div=true -prec-sqrt=true"
mkdir -p ../../tools/bin
nvcc $FLAGS -DGOOM_TC_TRACE -c lmme_tc.cu -o /tmp/lmme_tc_trace.o
nvcc $FLAGS -DGOOM_L64_TRACE -c scan_long_tc.cu -o /tmp/scan_long_tc_trace.o
objs=$(ls build/*.o | grep -v "lmme_tc.o\|scan_long_tc.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/bin/libgoom_trace.so $objs /tmp/lmme_tc_trace.o /tmp/scan_long_tc_trace.o -lcudart -ldl
