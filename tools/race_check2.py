"""Per process: L0 ABC and a given (level, variant) on cfg4 vs torch.einsum; where are the wrong elements?"""
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
import paper_1704_03092_b200 as stc  # noqa: E402
from perf_probe import CONFIGS, dev_tensor  # noqa: E402

name, level, variant = sys.argv[1], int(sys.argv[2]), sys.argv[3]
spec = stc.parse_benchmark_line(CONFIGS[name][0])
a = dev_tensor(spec.tensor_extents(spec.labels_a), 1)
b = dev_tensor(spec.tensor_extents(spec.labels_b), 2)
c0 = dev_tensor(spec.tensor_extents(spec.labels_c), 3)
ext = lambda t: torch.as_strided(t.data, t.extents, t.strides, t.base_offset)
gold = ext(c0) + torch.einsum(f"{spec.labels_a},{spec.labels_b}->{spec.labels_c}", ext(a), ext(b))
for lv, var in ((0, "abc"), (level, variant)):
    c = stc.DenseTensor(c0.extents, c0.strides, c0.data.clone())
    stc.contract(spec, a, b, c, lv, var)
    d = (ext(c) - gold).abs()
    err = (torch.linalg.vector_norm(ext(c) - gold) / torch.linalg.vector_norm(gold)).item()
    bad = torch.nonzero(d > 1e-9 * gold.abs().max())
    msg = f"L{lv} {var}: rel err {err:.3e}, wrong elements {bad.shape[0]}"
    if bad.shape[0]:
        for ax, l in enumerate(spec.labels_c):
            vals = torch.unique(bad[:, ax])
            msg += f" | {l}: {vals.numel()} values {vals[:6].tolist()}"
    print(msg, flush=True)
