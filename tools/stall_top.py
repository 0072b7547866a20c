"""Top stalled SASS instructions from an ncu source-page CSV (--page source --csv --print-source sass)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
st = [k for k in h if k.startswith('stall_') and 'Not Issued' not in k]
body = rows[2:]
tot = sum(int(r[idx['Warp Stall Sampling (All Samples)']] or 0) for r in body)
print('total samples', tot)
agg = {}
for n, r in enumerate(body):
    s = int(r[idx['Warp Stall Sampling (All Samples)']] or 0)
    agg[n] = s
top = sorted(agg, key=lambda n: -agg[n])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]
for n in sorted(top):
    r = body[n]
    parts = sorted(((int(float(r[idx[k]] or 0)), k[6:]) for k in st), reverse=True)[:3]
    print(f"{n:5d} {agg[n]*100/tot:5.2f}% {r[1].strip()[:60]:60s} {parts}")
