"""One contraction of a benchmark line against torch.einsum (row-major operands, optional storage offset).
Usage: python tools/repro_case.py "<line>" level variant [offset]"""
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_1704_03092_b200 as stc  # noqa: E402

line, level, variant = sys.argv[1], int(sys.argv[2]), sys.argv[3]
off = int(sys.argv[4]) if len(sys.argv) > 4 else 0
spec = stc.parse_benchmark_line(line)
gen = torch.Generator(device="cuda").manual_seed(7)


def tensor(labels, offset):
    e = spec.tensor_extents(labels)
    n = int(np.prod(e))
    flat = torch.rand(n + offset, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
    return torch.as_strided(flat, e, tuple(int(np.prod(e[i + 1:])) for i in range(len(e))), offset)


a, b, c = tensor(spec.labels_a, off), tensor(spec.labels_b, off), tensor(spec.labels_c, 0)
ref = c + torch.einsum(f"{spec.labels_a},{spec.labels_b}->{spec.labels_c}", a, b)
try:
    st = stc.contract(spec, a, b, c, level, variant)
    torch.cuda.synchronize()
    err = (torch.linalg.vector_norm(c - ref) / torch.linalg.vector_norm(ref)).item()
    print("OK " if err <= 1e-12 else "BAD", line, f"L{level} {variant} off {off} err {err:.3e} m,n,k={spec.n_i},{spec.n_j},{spec.n_p}",
          flush=True)
except RuntimeError as exc:
    print("CRASH", line, f"L{level} {variant} off {off}", str(exc)[:120], flush=True)
