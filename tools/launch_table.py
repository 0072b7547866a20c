"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): launches, total ms and
share per kernel.  Usage: python tools/launch_table.py launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    ns = float(r[14].replace(",", ""))
    tot[r[4]] += ns
    cnt[r[4]] += 1
allns = sum(tot.values())
print("| launches | ms | share | kernel |\n|---:|---:|---:|---|")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"| {cnt[k]} | {v / 1e6:.3f} | {100 * v / allns:.2f}% | `{k[:80]}` |")
