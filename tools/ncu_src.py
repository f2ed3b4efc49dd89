"""Summarise an `ncu --page source --csv --print-source sass` dump: per-SASS
instruction stall samples (the hot loop), for reading profiles here."""
import csv, sys

def main(path, top=80, min_samples=1):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    cols = ['stall_dispatch', 'stall_math', 'stall_wait', 'stall_short_sb', 'stall_long_sb',
            'stall_not_selected', 'stall_selected', 'stall_branch_resolving', 'stall_mio', 'stall_lg', 'stall_barrier']
    out = []
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        try:
            s = int(r[ix['Warp Stall Sampling (All Samples)']] or 0)
        except ValueError:
            continue
        out.append((r[ix['Address']], r[ix['Source']], s, {c: r[ix[c]] for c in cols if c in ix}))
    tot = sum(o[2] for o in out) or 1
    for a, src, s, d in out:
        if s >= min_samples:
            extra = ' '.join(f"{k[6:]}={v}" for k, v in d.items() if v not in ('0', ''))
            print(f"{a:>6} {s*100.0/tot:5.1f}% {src[:70]:70s} {extra}")

if __name__ == '__main__':
    main(sys.argv[1], min_samples=int(sys.argv[2]) if len(sys.argv) > 2 else 1)
