"""Source lines of the local-memory spills near DMMAs (distance < 40 instructions) of one kernel.
Usage: python tools/spill_near.py build/stc_fused.o <kernel-name-substring>"""
import collections
import os
import re
import subprocess
import sys
import tempfile

obj, pat = sys.argv[1], sys.argv[2]
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
parts = re.split(r"\n\s*\.text\.(\S+):", txt)
for i in range(1, len(parts), 2):
    name, body = parts[i], parts[i + 1]
    if pat not in name:
        continue
    ins, cur = [], None
    for line in body.split("\n"):
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        if re.search(r"/\*[0-9a-f]{4,}\*/", line):
            ins.append((cur, line.strip()))
    dmma = [k for k, (_, l) in enumerate(ins) if "DMMA" in l]
    c = collections.Counter()
    for k, (src, l) in enumerate(ins):
        if re.search(r"\b(STL|LDL)", l) and min(abs(k - j) for j in dmma) < 40:
            c[src] += 1
    print(name, c.most_common(10))
