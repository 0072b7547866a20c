for P in ${PIECES:-1 2 4 8}; do STC_HOST_TRACE=1 STC_HOST_PIECES=$P python - <<'PY'
import sys, pathlib
sys.path.insert(0, "tools")
import numpy as np, torch
import paper_1704_03092_b200 as stc
from perf_probe import CONFIGS, row_major
spec = stc.parse_benchmark_line(CONFIGS["cfg2"][0])
def host(labels, seed):
    e = spec.tensor_extents(labels)
    d = torch.from_numpy(np.random.default_rng(seed).uniform(-1, 1, int(np.prod(e)))).pin_memory()
    return stc.DenseTensor(e, row_major(e), d)
a, b, c = host(spec.labels_a, 1), host(spec.labels_b, 2), host(spec.labels_c, 3)
for _ in range(3):
    stc.contract(spec, a, b, c, 2, "abc")
x = torch.from_numpy(np.zeros(402653184 // 8)).pin_memory(); y = torch.empty_like(x, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    e0.record(); y.copy_(x, non_blocking=True); e1.record(); e1.synchronize()
print("plain H2D 402 MB:", e0.elapsed_time(e1), "ms", 402653184 / e0.elapsed_time(e1) / 1e6, "GB/s", file=sys.stderr)
for _ in range(2):
    e0.record(); x.copy_(y, non_blocking=True); e1.record(); e1.synchronize()
print("plain D2H 402 MB:", e0.elapsed_time(e1), "ms", file=sys.stderr)
PY
done
