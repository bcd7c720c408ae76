#!/bin/bash
# Builds libktg.so with extra -D flags into variants/<name>/ (git-ignored) for
# A/B runs through KTG_LIB_DIR: scripts/build_variant.sh <name> [-DFOO=1 ...]
set -e
name=$1; shift
d=variants/$name
mkdir -p $d
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  -Xptxas -v --expt-relaxed-constexpr "$@" -shared -o $d/libktg.so paper_2009_07929_b200/csrc/ktg_engine.cu -lcudart \
  2> $d/ptxas.log || (cat $d/ptxas.log; false)
cp paper_2009_07929_b200/lib/libktg_graph.so $d/ 2>/dev/null || true
grep -A1 "k_support_a22ILb0" $d/ptxas.log | grep -o "Used [0-9]* registers.*" || true
