"""BASELINE cfg3 shape sweep on one B200: Z[a,b,i,j] = sum_{e,f} W[a,b,e,f] T[e,f,i,j],
N_e = N_f = 64, N_a = N_b in {16, 32, 64, 128, 256}.

Two readings: "literal" N_i = N_j = 16384 / N_a (m*n = 2^28, 2.2 TFLOP per
point) and "2^24" N_i = N_j = 4096 / N_a (m*n = 2^24, 137 GFLOP per point).  Device-resident
operands, uniform[-1,1]; best of 3 timed calls after a warm-up.

Usage: python tools/cfg3_sweep.py [levels...]   (default 1 2)
"""

import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
import paper_1704_03092_b200 as stc  # noqa: E402
from perf_probe import dev_tensor  # noqa: E402


def main(levels):
    for reading, top in (("2^24", 4096), ("literal", 16384)):
        for na in (16, 32, 64, 128, 256):
            ni = top // na
            line = f"abij abef efij & a:{na};b:{na};i:{ni};j:{ni};e:64;f:64;"
            spec = stc.parse_benchmark_line(line)
            a = dev_tensor(spec.tensor_extents(spec.labels_a), 1)
            b = dev_tensor(spec.tensor_extents(spec.labels_b), 2)
            c = dev_tensor(spec.tensor_extents(spec.labels_c), 3, zero=True)
            flops = 2.0 * spec.n_i * spec.n_j * spec.n_p
            for level in levels:
                stc.contract(spec, a, b, c, level, "abc")
                best = min(stc.contract(spec, a, b, c, level, "abc").device_seconds for _ in range(3))
                print(f"cfg3 {reading:7s} N_a={na:3d} N_i={ni:4d} m={spec.n_i:6d} n={spec.n_j:8d} k={spec.n_p} "
                      f"L{level} ABC {best * 1e3:9.3f} ms  eff {flops / best / 1e12:6.2f} TF/s "
                      f"({100 * flops / best / 1e12 / 37.0:5.1f}% of 37.0)", flush=True)
            del a, b, c
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main([int(x) for x in sys.argv[1:]] or [1, 2])
