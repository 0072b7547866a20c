"""Repeat one contraction N times in one process against torch.einsum; count wrong runs.
Usage: python tools/race_check3.py config level variant reps"""
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
import paper_1704_03092_b200 as stc  # noqa: E402
from perf_probe import CONFIGS, dev_tensor  # noqa: E402

name, level, variant, reps = sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
spec = stc.parse_benchmark_line(CONFIGS[name][0])
a = dev_tensor(spec.tensor_extents(spec.labels_a), 1)
b = dev_tensor(spec.tensor_extents(spec.labels_b), 2)
c0 = dev_tensor(spec.tensor_extents(spec.labels_c), 3)
ext = lambda t: torch.as_strided(t.data, t.extents, t.strides, t.base_offset)
gold = ext(c0) + torch.einsum(f"{spec.labels_a},{spec.labels_b}->{spec.labels_c}", ext(a), ext(b))
bad = 0
for r in range(reps):
    c = stc.DenseTensor(c0.extents, c0.strides, c0.data.clone())
    stc.contract(spec, a, b, c, level, variant, allow_deep=level > 2)
    err = (torch.linalg.vector_norm(ext(c) - gold) / torch.linalg.vector_norm(gold)).item()
    bad += err > 1e-12
print(f"{name} L{level} {variant}: {reps} runs, {bad} wrong", flush=True)
