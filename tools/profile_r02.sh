#!/bin/bash
# Round-2 profile pass on one B200 (run under gpurun from the repo root):
#   1. bench line (no BO / render / CPU baseline: the kernels only)
#   2. launch list of one step: ncu --metrics gpu__time_duration.sum (cold, serialised)
#   3. one `ncu --set full` capture of k_vis_tiles and of k_depth_pairs
# Each ncu command runs only after the same command exited 0 without ncu.
set -u
OUT=gpurun_out/${1:-r02}
mkdir -p $OUT
ARGS="--steps 3 --warmup 3 --no-cpu-baseline --no-bo --e2e-steps 1 --render 0 --no-dense-ref"
python bench.py $ARGS > $OUT/bench.json 2> $OUT/bench.err || { echo "bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-bo --e2e-steps 1 --render 0 --no-dense-ref \
    > $OUT/ncu_launches.log 2>&1
for K in k_vis_tiles k_depth_pairs; do
  ncu --set full --import-source on --clock-control none -k regex:$K -s 3 -c 1 -o $OUT/$K \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-bo --e2e-steps 1 --render 0 --no-dense-ref \
      > $OUT/ncu_$K.log 2>&1
done
echo done
