"""Time one config under several STC_* environment settings (device time, best of 3):
python tools/env_probe.py "<benchmark line>" level variant "K=V,K=V" ["K=V" ...]"""
import os
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_1704_03092_b200 as stc  # noqa: E402
from paper_1704_03092_b200.synth import row_major, uniform_tensor  # noqa: E402

line, level, variant = sys.argv[1], int(sys.argv[2]), sys.argv[3]
spec = stc.parse_benchmark_line(line)
dev = torch.device("cuda", 0)
a = uniform_tensor(1, spec.tensor_extents(spec.labels_a), dev)
b = uniform_tensor(2, spec.tensor_extents(spec.labels_b), dev)
ec = spec.tensor_extents(spec.labels_c)
c = stc.DenseTensor(ec, row_major(ec), torch.zeros(int(np.prod(ec)), dtype=torch.float64, device=dev))
flops = 2.0 * spec.n_i * spec.n_j * spec.n_p
for combo in sys.argv[4:]:
    env = dict(kv.split("=") for kv in combo.split(",") if kv)
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    info = stc.describe_plan(spec, a, b, c, level, variant)
    stc.contract(spec, a, b, c, level, variant)
    best = min(stc.contract(spec, a, b, c, level, variant).device_seconds for _ in range(3))
    print(f"{combo:40s} {best * 1e3:9.3f} ms  {flops / best / 1e12:6.2f} TF/s  ticketed={info['ticketed']} "
          f"presum={info['presum']} pack={info['need_pack']} cboxes={info['c_boxes']}", flush=True)
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
