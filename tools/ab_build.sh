#!/bin/bash
# Build liblobe.so variants for an A/B timing run on the GPU box (tunelib/ is
# git-ignored but travels with gpurun). Usage:
#   tools/ab_build.sh <name> [<git-rev>]   -- kernels of <git-rev> (default: the working tree)
# then LOBE_LIB=tunelib/liblobe_<name>.so python tools/eval_time.py ...
set -eu
NAME=$1; REV=${2:-}
D=tunelib/$NAME; mkdir -p $D
C=paper_2510_01767_b200/csrc
for f in lobe_kernels.cu lobe_api.cpp lobe_bo.cpp lobe_comm.cpp lobe_internal.h lobe_comm.h; do
  if [ -n "$REV" ]; then git show $REV:$C/$f > $D/$f; else cp $C/$f $D/$f; fi
done
mkdir -p $D/include; cp include/lobe.h $D/include/ 2>/dev/null || true
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a"
$NV -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off -I include -c $D/lobe_kernels.cu -o $D/k.o
for f in lobe_api lobe_bo lobe_comm; do
  g++ -O2 -std=c++17 -fPIC -ffp-contract=off -fno-fast-math -Wall -Wno-unused-function -I /usr/local/cuda/include -I include -c $D/$f.cpp -o $D/$f.o
done
$NV -shared -o tunelib/liblobe_$NAME.so $D/k.o $D/lobe_api.o $D/lobe_bo.o $D/lobe_comm.o -ldl
echo tunelib/liblobe_$NAME.so
