"""Per-kernel times of the last bench step in an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file <csv> python bench.py ...`):
cold, serialised launches; for reading kernel shares here, never a bench value."""
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ix = {k: j for j, k in enumerate(h)}
    data = [r for r in rows[start + 1:] if len(r) == len(h) and r[ix["Metric Name"]] == "gpu__time_duration.sum"]
    names = [r[ix["Kernel Name"]] for r in data]
    last = max(i for i, n in enumerate(names) if "k_prep_raw" in n)
    tot = 0.0
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    for r in data[last:]:
        t = float(r[ix["Metric Value"]].replace(",", "")) * scale[r[ix["Metric Unit"]]]
        tot += t
        print(f"{t:9.1f} us  {r[ix['Kernel Name']][:70]}")
    print(f"total {tot:.1f} us")


if __name__ == "__main__":
    main(sys.argv[1])
