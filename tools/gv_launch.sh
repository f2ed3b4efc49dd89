mkdir -p gpurun_out/$1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$1/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-bo --e2e-steps 1 --render 0 --no-dense-ref > gpurun_out/$1/ncu_launches.log 2>&1
python tools/launch_summary.py gpurun_out/$1/launches.csv
