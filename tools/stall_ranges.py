"""Aggregate ncu stall reasons over SASS line ranges split at USETMAXREG (producer / consumer)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; idx = {k: i for i, k in enumerate(h)}
body = rows[2:]
st = [k for k in h if k.startswith('stall_') and 'Not Issued' not in k]
marks = [n for n, r in enumerate(body) if 'SETMAXREG' in r[1]]
print('setmaxreg at', marks)
bounds = [0] + marks + [len(body)]
for a, b in zip(bounds, bounds[1:]):
    tot = {k: 0 for k in st}
    ninst = 0
    for r in body[a:b]:
        for k in st:
            tot[k] += int(float(r[idx[k]] or 0))
        ninst += int(float(r[idx['Instructions Executed']] or 0))
    s = sum(tot.values())
    print(f'lines {a}-{b}: samples {s} warp-instr {ninst}')
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:8]:
        print(f'   {k:28s} {v:8d} {100*v/max(s,1):5.1f}%')
