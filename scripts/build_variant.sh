#!/bin/bash
# Build an A/B variant of the engine: ablbuild/ab/lib_<NAME>.so from the
# current sources with extra nvcc flags (e.g. -DSSQA_EPI_V=0).  Used only by
# scripts/gpu_ab.sh; never by the tests or the bench.
#   scripts/build_variant.sh NAME [-DFLAG=V ...]
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
mkdir -p build/ab ablbuild/ab
python paper_2302_12454_b200/build.py > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -Iinclude -Ipaper_2302_12454_b200/csrc "$@" \
  -c paper_2302_12454_b200/csrc/sweep_tc.cu -o build/ab/sweep_tc_$NAME.o
objs=$(ls build/obj/*.o | grep -v sweep_tc)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ablbuild/ab/lib_$NAME.so \
  build/ab/sweep_tc_$NAME.o $objs -lcuda
echo ablbuild/ab/lib_$NAME.so
