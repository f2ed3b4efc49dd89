"""Summarise an `ncu --set full` capture (.ncu-rep) into a small JSON for
profiles/: duration, DRAM bytes, pipe / issue utilisation, occupancy,
instruction count. bench.py reads profiles/r02_vis_tiles_ncu.json into its
roofline line (config / world identify the capture's workload).

python tools/ncu_summary.py <rep> <out.json> --config matrixcity --kernel k_vis_tiles --command "..."
"""
import argparse
import csv
import io
import json
import subprocess

METRICS = {
    "duration_ms": ("gpu__time_duration.sum", 1.0),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "fma_pipe_active_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "alu_pipe_active_pct": ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "fma_inst_pct": ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1.0),
    "alu_inst_pct": ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "warp_instructions": ("smsp__inst_executed.sum", 1.0),
    "sm_clock_ghz": ("sm__cycles_elapsed.avg.per_second", 1.0),
    "registers_per_thread": ("launch__registers_per_thread", 1.0),
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TIME_TO_MS = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--config", default="matrixcity")
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--command", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, v = rows[0], rows[1], rows[2]
    out = {"config": a.config, "world": 1, "kernel": a.kernel, "capture": a.command,
           "source": "ncu --set full --clock-control none (cold, serialised; one launch)"}
    for key, (m, _) in METRICS.items():
        if m in h:
            i = h.index(m)
            val = float(v[i].replace(",", ""))
            if key.startswith("dram_"):
                val *= SCALE.get(units[i], 1)
            if key == "duration_ms":  # ncu picks the unit per report
                val *= TIME_TO_MS.get(units[i], 1.0)
            out[key] = val
    if "dram_read_bytes" in out and "dram_write_bytes" in out:
        out["dram_bytes_per_launch"] = out["dram_read_bytes"] + out["dram_write_bytes"]
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
