"""Sweep: default plan vs forced pre-summed operands (STC_PRESUM_OPS=1) vs in-kernel sums (=0)
over the BASELINE configs; best-of-3 device time, effective TF/s, and whether the three
results are bitwise equal.  Usage: python tools/presum_sweep.py [names...]
"""

import os
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_1704_03092_b200 as stc  # noqa: E402
from paper_1704_03092_b200.synth import row_major, uniform_tensor  # noqa: E402

R = [(1, "abc"), (2, "abc"), (1, "ab"), (2, "ab"), (1, "naive"), (2, "naive")]
CONFIGS = {
    "cfg1": ("abij abef efij & a:24;b:24;i:24;j:24;e:24;f:24;", R),
    "cfg2": ("aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;", R),
    "cfg4": ("abcij eafbc ifje & a:50;b:7;c:13;i:70;j:45;e:90;f:33;", R),
    "bar": ("abij abef efij & a:128;b:128;i:128;j:128;e:128;f:128;", [(1, "abc"), (2, "abc"), (2, "ab")]),
    "cfg5s8": ("abcijk abcefg efgijk & a:32;b:32;c:32;i:4;j:32;k:32;e:32;f:32;g:32;", [(1, "abc"), (2, "abc")]),
}
for na in (16, 32, 64, 128, 256):
    CONFIGS[f"c3s{na}"] = (f"abij abef efij & a:{na};b:{na};i:{4096 // na};j:{4096 // na};e:64;f:64;",
                           [(1, "abc"), (2, "abc")])
CONFIGS["c3l16"] = ("abij abef efij & a:16;b:16;i:1024;j:1024;e:64;f:64;", [(1, "abc"), (2, "abc")])
CONFIGS["c3l256"] = ("abij abef efij & a:256;b:256;i:64;j:64;e:64;f:64;", [(1, "abc"), (2, "abc")])


def timed(spec, a, b, c, level, variant):
    stc.contract(spec, a, b, c, level, variant)
    best = 1e30
    for _ in range(3):
        c.data.zero_()
        st = stc.contract(spec, a, b, c, level, variant)
        best = min(best, st.device_seconds)
    return best, c.data.clone()


def main(names):
    dev = torch.device("cuda", 0)
    for name in names:
        line, runs = CONFIGS[name]
        spec = stc.parse_benchmark_line(line)
        a = uniform_tensor(1, spec.tensor_extents(spec.labels_a), dev)
        b = uniform_tensor(2, spec.tensor_extents(spec.labels_b), dev)
        ec = spec.tensor_extents(spec.labels_c)
        c = stc.DenseTensor(ec, row_major(ec), torch.zeros(int(np.prod(ec)), dtype=torch.float64, device=dev))
        flops = 2.0 * spec.n_i * spec.n_j * spec.n_p
        for level, variant in runs:
            res = {}
            for mode in (None, "0", "1"):
                if mode is None:
                    os.environ.pop("STC_PRESUM_OPS", None)
                else:
                    os.environ["STC_PRESUM_OPS"] = mode
                info = stc.describe_plan(spec, a, b, c, level, variant)
                t, out = timed(spec, a, b, c, level, variant)
                res[mode] = (t, out, info["presum"], info["ticketed"])
            os.environ.pop("STC_PRESUM_OPS", None)
            same = torch.equal(res[None][1], res["0"][1]) and torch.equal(res[None][1], res["1"][1])
            cells = "  ".join(f"{'def' if m is None else 'ps' + m}:{flops / res[m][0] / 1e12:6.2f}"
                              f"{'*' if res[m][2] else ' '}" for m in (None, "0", "1"))
            print(f"{name:7s} L{level} {variant:5s} {cells}  ticketed={res[None][3]}  bitwise={same}", flush=True)
            del res
        del a, b, c
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1:] or list(CONFIGS))
