"""Pre-summed operands (STC_PRESUM_OPS=1) vs in-kernel sums (=0): timing and bitwise check.

Usage: python tools/presum_probe.py [names...]  (cfg2 bar cfg5 cfg5s8 cfg2L1 barL1 cfg3l)
"""

import os
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_1704_03092_b200 as stc  # noqa: E402
from paper_1704_03092_b200.synth import row_major, uniform_tensor  # noqa: E402

CONFIGS = {
    "cfg2": ("aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;", 2),
    "cfg2L1": ("aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;", 1),
    "cfg2h": ("aibj eafb jfie & a:32;b:64;i:64;j:64;e:64;f:64;", 2),
    "b8k": ("abij abef efij & a:64;b:128;i:64;j:128;e:64;f:128;", 2),
    "bar": ("abij abef efij & a:128;b:128;i:128;j:128;e:128;f:128;", 2),
    "barL1": ("abij abef efij & a:128;b:128;i:128;j:128;e:128;f:128;", 1),
    "cfg5s8": ("abcijk abcefg efgijk & a:32;b:32;c:32;i:4;j:32;k:32;e:32;f:32;g:32;", 2),
    "cfg5": ("abcijk abcefg efgijk & a:32;b:32;c:32;i:32;j:32;k:32;e:32;f:32;g:32;", 2),
    "cfg3l": ("abij abef efij & a:64;b:64;i:256;j:256;e:64;f:64;", 2),
}


def run(name, reps):
    line, level = CONFIGS[name]
    spec = stc.parse_benchmark_line(line)
    dev = torch.device("cuda", 0)
    a = uniform_tensor(1, spec.tensor_extents(spec.labels_a), dev)
    b = uniform_tensor(2, spec.tensor_extents(spec.labels_b), dev)
    ec = spec.tensor_extents(spec.labels_c)
    flops = 2.0 * spec.n_i * spec.n_j * spec.n_p
    out = {}
    for mode in ("0", "1"):
        os.environ["STC_PRESUM_OPS"] = mode
        c = stc.DenseTensor(ec, row_major(ec), torch.zeros(int(np.prod(ec)), dtype=torch.float64, device=dev))
        stc.contract(spec, a, b, c, level, "abc")
        first = c.data.clone()
        ts, ks = [], []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0.record()  # torch creates the cudaEvent_t lazily, on first record
            k1.record()
            c.data.zero_()
            torch.cuda.synchronize()
            e0.record()
            stc.contract(spec, a, b, c, level, "abc", kernel_events=(k0, k1), synchronize=False)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
            ks.append(k0.elapsed_time(k1))
        same = bool(torch.equal(c.data, first))
        out[mode] = (min(ts), min(ks), c.data.clone(), same)
        print(f"{name:7s} L{level} presum={mode}  {min(ts):9.3f} ms  eff {flops / min(ts) / 1e9:6.2f} TF/s  "
              f"fused {min(ks):9.3f} ms ({flops / min(ks) / 1e9:6.2f})  rerun-bitwise {same}", flush=True)
        del c
    print(f"{name:7s} bitwise presum==in-kernel: {bool(torch.equal(out['0'][2], out['1'][2]))}", flush=True)
    del a, b, out
    torch.cuda.empty_cache()


if __name__ == "__main__":
    names = sys.argv[1:] or ["cfg2", "bar"]
    for n in names:
        run(n, 2 if n == "cfg5" else 5)
