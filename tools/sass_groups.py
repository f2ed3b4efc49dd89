"""Read an `ncu --page source --csv --print-source sass` export: SASS grouped into
runs of equal execution count (basic blocks of the hot loops), with the warp
instructions each run accounts for and its stall samples.

python tools/sass_groups.py <k_sass.csv> [--dump START END]   (address suffixes)"""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    out = []
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        out.append((r[ix['Address']][-5:], r[ix['Source']].strip(), int(r[ix['Instructions Executed']] or 0),
                    int(r[ix['Warp Stall Sampling (All Samples)']] or 0)))
    return out


def groups(out):
    tot = sum(o[2] for o in out)
    print('total warp instructions', tot)
    grp = []

    def flush():
        if grp and grp[0][2] * len(grp) > tot * 0.002:
            e = grp[0][2]
            ops = ' | '.join(g[1].split()[0] if not g[1].startswith('@') else ' '.join(g[1].split()[:2]) for g in grp)
            print(f"{grp[0][0]}-{grp[-1][0]} n={len(grp):3d} exec={e:>10d} {e * len(grp) / tot * 100:5.1f}% "
                  f"stall={sum(g[3] for g in grp)}  {ops[:220]}")
    for o in out:
        if grp and o[2] == grp[0][2]:
            grp.append(o)
        else:
            flush()
            grp[:] = [o]
    flush()


if __name__ == '__main__':
    out = load(sys.argv[1])
    if '--dump' in sys.argv:
        a, b = sys.argv[sys.argv.index('--dump') + 1:sys.argv.index('--dump') + 3]
        on = False
        for o in out:
            on = on or o[0] == a
            if on:
                print(o[0], f"{o[2]:>10d} {o[3]:>6d}", o[1])
            if o[0] == b:
                break
    else:
        groups(out)
