"""SASS instruction histogram of the library's kernels (cuobjdump of the built .so):
python tools/sass_hist.py [kernel-substring ...] > profiles/rNN_sass_histogram.txt"""
import collections
import pathlib
import re
import subprocess
import sys

SO = pathlib.Path(__file__).resolve().parents[1] / "paper_1704_03092_b200" / "libstc_b200.so"
KEYS = ["DMMA", "DFMA", "DADD", "DMUL", "UTMALDG", "UTMAREDG", "UTMASTG", "UBLKCP", "LDS", "STS", "LDG", "STG",
        "LDGSTS", "LDL", "STL", "SYNCS", "BAR", "SHFL"]
pats = sys.argv[1:] or ["k_strassen_fused", "k_presum", "k_accumulate", "k_strassen_gemm"]
txt = subprocess.run(["cuobjdump", "-sass", str(SO)], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", txt)
print(f"# SASS histogram of {SO.name} (cuobjdump -sass), one row per kernel instance")
print("| kernel | " + " | ".join(KEYS) + " |")
print("|---|" + "---:|" * len(KEYS))
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if not any(p in name for p in pats):
        continue
    ops = collections.Counter()
    for line in f.split("\n"):
        m = re.search(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            ops[m.group(1)] += 1
    row = [sum(v for k, v in ops.items() if k == key or k.startswith(key + ".")) for key in KEYS]
    short = re.sub(r"^_ZN3stc", "", name)[:70]
    print(f"| `{short}` | " + " | ".join(str(x) for x in row) + " |")
