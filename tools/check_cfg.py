"""Full-size correctness check of the B200 path against a torch.einsum fp64 classical contraction.

Usage: python tools/check_cfg.py cfg2 [level variant ...]   (default: the config's perf_probe runs)
Prints the normwise relative error ||C - C_ref|| / ||C_ref|| and which staging path ran
(fast_blocks > 0: TMA box loads; slow_blocks: cp.async gather).
"""

import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
import paper_1704_03092_b200 as stc  # noqa: E402
from perf_probe import CONFIGS, dev_tensor  # noqa: E402


def main(argv):
    name = argv[0]
    line, runs = CONFIGS[name]
    if len(argv) > 1:
        runs = [(int(argv[i]), argv[i + 1]) for i in range(1, len(argv), 2)]
    spec = stc.parse_benchmark_line(line)
    a = dev_tensor(spec.tensor_extents(spec.labels_a), 1)
    b = dev_tensor(spec.tensor_extents(spec.labels_b), 2)
    ta = a.data.view(a.extents)
    tb = b.data.view(b.extents)
    ref = torch.einsum(f"{spec.labels_a},{spec.labels_b}->{spec.labels_c}", ta, tb)
    nref = torch.linalg.vector_norm(ref).item()
    for level, variant in runs:
        c = dev_tensor(spec.tensor_extents(spec.labels_c), 3, zero=True)
        st = stc.contract(spec, a, b, c, level, variant)
        err = torch.linalg.vector_norm(c.data.view(c.extents) - ref).item() / nref
        print(f"{name} L{level} {variant:5s} rel_err {err:.3e}  fast_blocks {st.fast_blocks}  slow_blocks {st.slow_blocks}"
              f"  {'OK' if err <= 1e-10 else 'FAIL'}", flush=True)
        del c


if __name__ == "__main__":
    main(sys.argv[1:])
