"""One warm contract() with extra contract() options (for ncu captures):
python tools/one_call_opts.py <config> <level> <variant> [force_slow] [allow_deep]"""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
import torch  # noqa: E402

import paper_1704_03092_b200 as stc  # noqa: E402
from perf_probe import CONFIGS, dev_tensor  # noqa: E402

name, level, variant = sys.argv[1], int(sys.argv[2]), sys.argv[3]
opts = {o: True for o in sys.argv[4:]}
spec = stc.parse_benchmark_line(CONFIGS[name][0])
a = dev_tensor(spec.tensor_extents(spec.labels_a), 1)
b = dev_tensor(spec.tensor_extents(spec.labels_b), 2)
c = dev_tensor(spec.tensor_extents(spec.labels_c), 3, zero=True)
for _ in range(2):
    st = stc.contract(spec, a, b, c, level, variant, **opts)
torch.cuda.synchronize()
print(f"{name} L{level} {variant} {opts}: {st.device_seconds * 1e3:.3f} ms")
