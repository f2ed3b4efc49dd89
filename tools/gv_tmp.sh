D=gpurun_out/$1; mkdir -p $D
python -m pytest tests -x -q -m gpu > $D/gpu.log 2>&1; echo "gpu tests rc=$?"; tail -1 $D/gpu.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-bo --render 0 --no-dense-ref --e2e-steps 5 > $D/b.json 2> $D/b.err
python -c "import json;d=json.loads(open('$D/b.json').read().strip().splitlines()[-1]);r=d['roofline'];print('step',round(d['ms_per_step'],3),'vis',round(d['t_vis_ms_max_over_ranks'],3),'frac',round(r['frac'],3),'issued',round(r['issued']['frac'],3), 'e2e', round(d['e2e']['ms_per_step'],3))"
