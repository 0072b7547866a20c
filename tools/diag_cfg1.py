import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import oracle
import paper_1704_03092_b200 as stc
line = sys.argv[1] if len(sys.argv) > 1 else "abij abef efij & a:24;b:24;i:24;j:24;e:24;f:24;"
spec = stc.parse_benchmark_line(line)
def rm(ext):
    out, run = [], 1
    for e in reversed(ext): out.append(run); run *= e
    return tuple(reversed(out))
def T(labels, seed):
    ext = spec.tensor_extents(labels)
    return stc.DenseTensor(ext, rm(ext), np.random.default_rng(seed).uniform(-1, 1, int(np.prod(ext))))
a, b = T(spec.labels_a, 7), T(spec.labels_b, 8)
c0 = stc.DenseTensor(spec.tensor_extents(spec.labels_c), rm(spec.tensor_extents(spec.labels_c)), np.zeros(spec.n_i * spec.n_j))
ref = c0.copy(); oracle.contract_reference(spec, a, b, ref, threads=8)
for level in (0, 1, 2):
    for variant in ("abc", "ab", "naive"):
        for kw in ({}, {"force_slow": True}, {"reference_tiling": True}, {"force_slow": True, "reference_tiling": True}):
            c = c0.copy()
            stc.contract(spec, a, b, c, level, variant, **kw)
            print(level, variant, kw, f"{oracle.relative_error(c, ref):.3e}", flush=True)
