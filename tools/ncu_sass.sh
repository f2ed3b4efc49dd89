#!/bin/bash
# One `ncu --set full` capture per kernel named on the command line (bench step,
# MatrixCity), exported as SASS-level source CSV + raw metrics for reading here
# (tools/sass_groups.py). Run under gpurun from the repo root:
#   tools/ncu_sass.sh <outdir> k_vis_tiles k_hist ...
set -u
OUT=gpurun_out/$1; shift
mkdir -p $OUT
A="--steps 1 --warmup 3 --no-cpu-baseline --no-bo --e2e-steps 1 --render 0 --no-dense-ref"
for K in "$@"; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$K -s 3 -c 1 -o $OUT/$K \
      python bench.py $A > $OUT/ncu_$K.log 2>&1
  ncu -i $OUT/$K.ncu-rep --page source --csv --print-source sass > $OUT/${K}_sass.csv 2>&1
  ncu -i $OUT/$K.ncu-rep --page raw --csv > $OUT/${K}_raw.csv 2>&1
done
echo done
