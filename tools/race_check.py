"""Run one contraction repeatedly on the same inputs; report results that differ (races).
Usage: python tools/race_check.py cfg4 1 ab [reps] (configs of tools/perf_probe.py)"""
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
import paper_1704_03092_b200 as stc  # noqa: E402
from perf_probe import CONFIGS, dev_tensor  # noqa: E402

name, level, variant = sys.argv[1], int(sys.argv[2]), sys.argv[3]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
spec = stc.parse_benchmark_line(CONFIGS[name][0])
a = dev_tensor(spec.tensor_extents(spec.labels_a), 1)
b = dev_tensor(spec.tensor_extents(spec.labels_b), 2)
c0 = dev_tensor(spec.tensor_extents(spec.labels_c), 3)
ref = stc.DenseTensor(c0.extents, c0.strides, c0.data.clone())
stc.contract(spec, a, b, ref, 0, "abc")
first = None
bad = 0
for r in range(reps):
    c = stc.DenseTensor(c0.extents, c0.strides, c0.data.clone())
    stc.contract(spec, a, b, c, level, variant)
    err = stc.relative_error(c, ref)
    same = first is None or torch.equal(c.data, first)
    if first is None:
        first = c.data.clone()
    if err > 1e-12 or not same:
        bad += 1
        diff = (c.data - first).abs()
        idx = torch.nonzero(diff > 0)[:5].tolist() if not same else []
        print(f"rep {r}: rel err vs L0 {err:.3e}, bitwise same as rep 0: {same}, first differing flat idx {idx}")
print(f"{name} L{level} {variant}: {reps} reps, {bad} bad")
