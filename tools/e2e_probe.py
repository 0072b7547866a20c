"""e2e probe: contract() on pinned host operands (cfg2 L2 ABC), wall time per call."""
import sys, time, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
import numpy as np, torch
import paper_1704_03092_b200 as stc
from perf_probe import CONFIGS, row_major
spec = stc.parse_benchmark_line(CONFIGS["cfg2"][0])
def host(labels, seed):
    e = spec.tensor_extents(labels)
    d = torch.from_numpy(np.random.default_rng(seed).uniform(-1, 1, int(np.prod(e)))).pin_memory()
    return stc.DenseTensor(e, row_major(e), d)
a, b, c = host(spec.labels_a, 1), host(spec.labels_b, 2), host(spec.labels_c, 3)
for _ in range(2):
    stc.contract(spec, a, b, c, 2, "abc")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    st = stc.contract(spec, a, b, c, 2, "abc")
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print(f"e2e {dt*1e3:.2f} ms/call  {2*4096**3/dt/1e9:.0f} GFLOP/s  (device {st.seconds*1e3:.2f} ms)")
