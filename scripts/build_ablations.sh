#!/bin/bash
# Build timing-ablation variants of the engine (never used by tests/bench):
#   build/abl/libssqa_abl<N>.so with -DSSQA_ABL=<N>
set -e
cd /root/repo
mkdir -p build/abl ablbuild
for A in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -Iinclude -Ipaper_2302_12454_b200/csrc -DSSQA_ABL=$(echo $A | cut -d_ -f1) $(echo $A | grep -q _r0 && echo -DSSQA_ENERGY_RED=0) -c paper_2302_12454_b200/csrc/sweep_tc.cu -o build/abl/sweep_tc_$A.o
  objs=$(ls build/obj/*.o | grep -v sweep_tc)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ablbuild/libssqa_abl$A.so build/abl/sweep_tc_$A.o $objs -lcuda
done
