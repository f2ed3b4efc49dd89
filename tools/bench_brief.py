"""One-screen summary of a bench.py JSON line (diagnosis while iterating)."""
import json
import sys

for path in sys.argv[1:]:
    d = json.loads(open(path).read().strip().splitlines()[-1])
    r = d["roofline"]
    ev = d.get("evaluation_roofline", {})
    dp = d.get("depth_roofline", {})
    print(f"{path}: step {d['ms_per_step']:.3f} ms  value {d['value']:.3e}  frac {r['frac']:.3f} "
          f"(issued {r.get('issued', {}).get('frac', 0):.3f})  t_vis {r['kernel_ms']:.3f} (cull {r['cull_ms']:.3f})  "
          f"eval {ev.get('ms', 0):.3f} (in step {ev.get('in_step_ms', 0):.3f})  a4 {dp.get('kernel_ms', 0):.3f} "
          f"(in step {dp.get('in_step_ms', 0):.3f})  engine {d.get('engine_eval_ms', 0):.3f}  "
          f"e2e {d['e2e']['ms_per_step']:.2f} ms  clocks {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
