#!/bin/bash
# Round-2 final measurement pass on one B200 (run under gpurun from the repo root):
# the default bench line, the other BASELINE configs, the anisotropic mode, the
# reference arm, then the launch list of one step and the ncu captures.
set -u
OUT=gpurun_out/final
mkdir -p $OUT/configs
python bench.py > $OUT/bench_mc.json 2> $OUT/bench_mc.err || echo "bench failed"
for c in rubble building residence; do
  python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-bo --render 0 > $OUT/configs/$c.json 2> $OUT/configs/$c.err
done
python bench.py --predicate aniso --steps 10 --warmup 3 --no-cpu-baseline --no-bo --render 0 > $OUT/configs/matrixcity_aniso.json 2> $OUT/configs/aniso.err
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-bo --e2e-steps 1 --render 0 --no-dense-ref"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py $ARGS > $OUT/ncu_launches.log 2>&1
for K in k_vis_tiles k_depth_pairs; do
  ncu --set full --import-source on --clock-control none -k regex:$K -s 3 -c 1 -o $OUT/$K python bench.py $ARGS > $OUT/ncu_$K.log 2>&1
done
echo done
