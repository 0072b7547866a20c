"""Run one warm contract() of a BASELINE config (for ncu captures): python tools/one_call.py cfg2 2 abc [reps]"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
import torch
import paper_1704_03092_b200 as stc
from perf_probe import CONFIGS, dev_tensor

name, level, variant = sys.argv[1], int(sys.argv[2]), sys.argv[3]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
spec = stc.parse_benchmark_line(CONFIGS[name][0])
a = dev_tensor(spec.tensor_extents(spec.labels_a), 1)
b = dev_tensor(spec.tensor_extents(spec.labels_b), 2)
c = dev_tensor(spec.tensor_extents(spec.labels_c), 3, zero=True)
for _ in range(reps):
    st = stc.contract(spec, a, b, c, level, variant)
torch.cuda.synchronize()
print(f"{name} L{level} {variant}: {st.device_seconds*1e3:.3f} ms eff {2.0*spec.n_i*spec.n_j*spec.n_p/st.device_seconds/1e12:.2f} TF/s")
