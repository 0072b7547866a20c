"""Quick performance probe of the B200 path on the BASELINE configs (device-resident inputs).

Usage: python tools/perf_probe.py [names...]   (names: cfg1 cfg2 cfg3 cfg4 bar)
Prints one line per (config, level, variant): best-of-N seconds, effective TFLOP/s.
"""

import pathlib
import sys
import time

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_1704_03092_b200 as stc  # noqa: E402

CONFIGS = {
    "cfg1": ("abij abef efij & a:24;b:24;i:24;j:24;e:24;f:24;", [(1, "abc"), (2, "abc"), (0, "abc"), (1, "ab"), (2, "ab")]),
    "cfg2": ("aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;", [(2, "abc"), (1, "abc"), (0, "abc"), (2, "ab"),
                                                                 (2, "naive")]),
    "cfg3a": ("abij abef efij & a:16;b:16;i:16;j:16;e:64;f:64;", [(1, "abc"), (2, "abc")]),
    "cfg3e": ("abij abef efij & a:256;b:256;i:16;j:16;e:64;f:64;", [(1, "abc"), (2, "abc")]),
    "cfg3m": ("abij abef efij & a:16;b:16;i:256;j:256;e:64;f:64;", [(1, "abc"), (2, "abc")]),
    "cfg4": ("abcij eafbc ifje & a:50;b:7;c:13;i:70;j:45;e:90;f:33;", [(1, "ab"), (1, "naive"), (2, "ab"),
                                                                       (2, "naive"), (2, "abc"), (0, "abc")]),
    "cfg2s": ("aibj eafb jfie & a:32;b:64;i:32;j:64;e:32;f:64;", [(2, "abc"), (1, "abc"), (0, "abc"), (2, "ab"),
                                                                  (2, "naive")]),
    # cfg2 pieces of the host pipeline (I bundle cut on a into 2 / 4 / 8)
    "cfg3l16": ("abij abef efij & a:16;b:16;i:1024;j:1024;e:64;f:64;", [(2, "abc")]),
    "cfg2h": ("aibj eafb jfie & a:32;b:64;i:64;j:64;e:64;f:64;", [(2, "abc"), (1, "abc")]),
    "cfg2q": ("aibj eafb jfie & a:16;b:64;i:64;j:64;e:64;f:64;", [(2, "abc"), (1, "abc"), (2, "ab"), (1, "ab")]),
    "cfg2e": ("aibj eafb jfie & a:8;b:64;i:64;j:64;e:64;f:64;", [(2, "abc"), (1, "abc")]),
    "cfg2L2": ("aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;", [(2, "abc")]),
    "barL2": ("abij abef efij & a:128;b:128;i:128;j:128;e:128;f:128;", [(2, "abc")]),
    "bar": ("abij abef efij & a:128;b:128;i:128;j:128;e:128;f:128;", [(2, "abc"), (1, "abc"), (0, "abc")]),
    # cfg5 per-GPU shards of the 8-GPU n-split (i: 32 / G), G = 8 and G = 1 (the full 32768^3)
    "cfg5s8": ("abcijk abcefg efgijk & a:32;b:32;c:32;i:4;j:32;k:32;e:32;f:32;g:32;", [(2, "abc"), (1, "abc")]),
    # cfg5 host-pipeline pieces: 4 x 8 grid (8192 x 4096) and 8 x 8 (4096 x 4096), k = 32768
    "cfg5p48": ("abcijk abcefg efgijk & a:8;b:32;c:32;i:4;j:32;k:32;e:32;f:32;g:32;", [(2, "abc")]),
    "cfg5p88": ("abcijk abcefg efgijk & a:4;b:32;c:32;i:4;j:32;k:32;e:32;f:32;g:32;", [(2, "abc")]),
    "cfg5v": ("abcijk abcefg efgijk & a:32;b:32;c:32;i:32;j:32;k:32;e:32;f:32;g:32;", [(2, "ab"), (2, "naive"),
                                                                                      (1, "abc"), (0, "abc")]),
    # three levels (allow_deep): pre-summed slots of 343 terms (k_presum<3>)
    "deep": ("abij abef efij & a:128;b:128;i:128;j:128;e:128;f:128;", [(3, "abc"), (3, "ab"), (3, "naive")]),
    "cfg5deep": ("abcijk abcefg efgijk & a:32;b:32;c:32;i:32;j:32;k:32;e:32;f:32;g:32;", [(3, "abc"), (3, "naive")]),
    "cfg2deep": ("aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;", [(3, "abc"), (3, "naive")]),
    "cfg5": ("abcijk abcefg efgijk & a:32;b:32;c:32;i:32;j:32;k:32;e:32;f:32;g:32;", [(2, "abc")]),
}


def row_major(ext):
    out, run = [], 1
    for e in reversed(ext):
        out.append(run)
        run *= e
    return tuple(reversed(out))


def dev_tensor(ext, seed, zero=False):
    n = int(np.prod(ext))
    if zero:
        data = torch.zeros(n, dtype=torch.float64, device="cuda")
    else:
        g = torch.Generator(device="cuda")
        g.manual_seed(seed)
        data = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    return stc.DenseTensor(ext, row_major(ext), data)


def main(names):
    for name in names:
        line, runs = CONFIGS[name]
        spec = stc.parse_benchmark_line(line)
        a = dev_tensor(spec.tensor_extents(spec.labels_a), 1)
        b = dev_tensor(spec.tensor_extents(spec.labels_b), 2)
        c = dev_tensor(spec.tensor_extents(spec.labels_c), 3, zero=True)
        for level, variant in runs:
            kw = {"allow_deep": True} if level > 2 else {}
            stc.contract(spec, a, b, c, level, variant, **kw)  # warm-up
            best = 1e30
            reps = 3
            for _ in range(reps):
                st = stc.contract(spec, a, b, c, level, variant, **kw)
                best = min(best, st.device_seconds)
            eff = 2.0 * spec.n_i * spec.n_j * spec.n_p / best / 1e12
            print(f"{name:6s} L{level} {variant:5s} m,n,k={spec.n_i},{spec.n_j},{spec.n_p}  {best * 1e3:9.3f} ms"
                  f"  eff {eff:7.2f} TF/s  executed {st.total_flops / best / 1e12:6.2f} TF/s  launches {st.kernel_launches}",
                  flush=True)
        del a, b, c
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg1", "cfg2", "cfg4", "bar"])
