"""e2e (pinned host operands) of a large config at several host-pipeline piece counts, with the
per-piece device timeline (STC_HOST_TRACE=1 prints it on stderr).
Usage: python tools/e2e_big.py "<benchmark line>" level variant setting...
(setting: default | N pieces | K=V,K=V environment, e.g. STC_HOST_GRID=8x8,STC_HOST_SHARE=0)"""
import os
import pathlib
import sys
import time

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_1704_03092_b200 as stc  # noqa: E402
from paper_1704_03092_b200.synth import row_major, uniform_tensor  # noqa: E402

line, level, variant = sys.argv[1], int(sys.argv[2]), sys.argv[3]
spec = stc.parse_benchmark_line(line)
dev = torch.device("cuda", 0)
flops = 2.0 * spec.n_i * spec.n_j * spec.n_p


def pinned(labels, seed):
    e = spec.tensor_extents(labels)
    t = uniform_tensor(seed, e, dev)
    h = torch.empty(t.data.numel(), dtype=torch.float64, pin_memory=True)
    h.copy_(t.data)
    del t
    torch.cuda.empty_cache()
    return stc.DenseTensor(e, row_major(e), h)


a, b = pinned(spec.labels_a, 1), pinned(spec.labels_b, 2)
ec = spec.tensor_extents(spec.labels_c)
c = stc.DenseTensor(ec, row_major(ec), torch.zeros(int(np.prod(ec)), dtype=torch.float64, pin_memory=True))
for p in sys.argv[4:]:
    env = dict(kv.split("=") for kv in p.split(",")) if "=" in p else ({} if p == "default" else {"STC_HOST_PIECES": p})
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    stc.contract(spec, a, b, c, level, variant)
    torch.cuda.synchronize()
    ts = []
    for _ in range(2):
        t0 = time.perf_counter()
        st = stc.contract(spec, a, b, c, level, variant)
        ts.append(time.perf_counter() - t0)
    dt = min(ts)
    print(f"pieces={p} ({st.pieces}): e2e {dt * 1e3:.1f} ms  {flops / dt / 1e12:.2f} TF/s  "
          f"device {st.device_seconds * 1e3:.1f} ms", flush=True)
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
