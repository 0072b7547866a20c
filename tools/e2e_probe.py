"""e2e probe: contract() on pinned host operands (cfg2 L2 ABC), wall time per call, for the
host pipeline at several piece counts (STC_HOST_PIECES) and the staged path (STC_HOST_PIPELINE=0).

Usage: python tools/e2e_probe.py [config] [level] [variant]
"""
import os, sys, time, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
import numpy as np, torch
import paper_1704_03092_b200 as stc
from perf_probe import CONFIGS, row_major

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
level = int(sys.argv[2]) if len(sys.argv) > 2 else 2
variant = sys.argv[3] if len(sys.argv) > 3 else "abc"
spec = stc.parse_benchmark_line(CONFIGS[name][0])
flops = 2.0 * spec.n_i * spec.n_j * spec.n_p


def host(labels, seed):
    e = spec.tensor_extents(labels)
    d = torch.from_numpy(np.random.default_rng(seed).uniform(-1, 1, int(np.prod(e)))).pin_memory()
    return stc.DenseTensor(e, row_major(e), d)


a, b, c = host(spec.labels_a, 1), host(spec.labels_b, 2), host(spec.labels_c, 3)
for env in ({"STC_HOST_PIPELINE": "0"}, {"STC_HOST_PIECES": "1"}, {"STC_HOST_PIECES": "2"}, {},
            {"STC_HOST_PIECES": "8"}, {"STC_HOST_PIECES": "16"}):
    os.environ.update(env)
    for _ in range(2):
        stc.contract(spec, a, b, c, level, variant)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        st = stc.contract(spec, a, b, c, level, variant)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"{name} L{level} {variant} {env or 'default'}: e2e {dt * 1e3:.2f} ms/call  {flops / dt / 1e9:.0f} GFLOP/s  "
          f"(call seconds {st.seconds * 1e3:.2f} ms, launches {st.kernel_launches})", flush=True)
    for k in env:
        del os.environ[k]
