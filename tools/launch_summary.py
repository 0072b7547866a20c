"""Summarise a launch-list csv (tools/launch_list.sh): the last call's library kernels."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
launches = {}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if "stc" not in d["Kernel Name"]:
            continue
        key = int(d["ID"])
        launches.setdefault(key, {"name": d["Kernel Name"].split("(")[0].replace("void ", "")})
        launches[key][d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
ids = sorted(launches)
half = ids[len(ids) // 2:]  # the second (warm) call
tot = sum(launches[i]["gpu__time_duration.sum"][0] for i in half)
print(f"| kernel | time | share | DRAM rd | DRAM wr |")
print("|---|---:|---:|---:|---:|")
for i in half:
    L = launches[i]
    t, u = L["gpu__time_duration.sum"]
    rd, ru = L.get("dram__bytes_read.sum", (0, ""))
    wr, wu = L.get("dram__bytes_write.sum", (0, ""))
    print(f"| `{L['name'][:48]}` | {t:.1f} {u} | {100 * t / tot:.1f}% | {rd:.3f} {ru} | {wr:.3f} {wu} |")
