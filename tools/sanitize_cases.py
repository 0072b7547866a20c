"""Small contractions covering every kernel path, for compute-sanitizer (one tool per run):

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_cases.py

* irregular layout with PAD quadrants (cfg4 pattern, small): L0 / L1 / L2 x ABC / AB / Naive
  (repacked operands, pre-summed slots, dense M + accumulate, load/add/store epilogue);
* box-regular layout (cfg2 pattern, 256 x 512 x 256): L1 / L2 ABC with in-kernel sums
  (summing warpgroup, TMA box loads, TMA reduce-add C epilogue, tickets) and with
  pre-summed slots; force_slow (the cp.async gather kernel);
* host operands (the piecewise host pipeline, 2 pieces).
Each result is checked against the CPU oracle (1e-12).
"""

import os
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
import paper_1704_03092_b200 as stc  # noqa: E402


def rm(e):
    return tuple(int(np.prod(e[i + 1:])) for i in range(len(e)))


def operands(spec, seed):
    def t(labels, s):
        e = spec.tensor_extents(labels)
        return stc.DenseTensor(e, rm(e), np.random.default_rng(s).uniform(-1, 1, int(np.prod(e))))
    return t(spec.labels_a, seed), t(spec.labels_b, seed + 1), t(spec.labels_c, seed + 2)


def check(spec, a, b, c0, level, variant, env=None, host=False, **kw):
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        ref = c0.copy()
        oracle.contract_reference(spec, a, b, ref)
        if host:
            c = c0.copy()
            stc.contract(spec, a, b, c, level, variant, **kw)
        else:
            c = c0.to_device()
            stc.contract(spec, a.to_device(), b.to_device(), c, level, variant, **kw)
            c = c.to_host()
        err = oracle.relative_error(c, ref)
        assert err <= 1e-12, (level, variant, env, err)
        print(f"ok L{level} {variant} {env or ''} {'host' if host else ''} {kw or ''} err {err:.1e}", flush=True)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def main():
    irr = stc.parse_benchmark_line("abcij eafbc ifje & a:10;b:7;c:13;i:14;j:9;e:18;f:11;")
    a, b, c0 = operands(irr, 1)
    for level in (0, 1, 2):
        for variant in ("abc", "ab", "naive"):
            check(irr, a, b, c0, level, variant)
    check(irr, a, b, c0, 2, "abc", {"STC_PRESUM_OPS": "1"})
    reg = stc.parse_benchmark_line("aibj eafb jfie & a:4;b:64;i:8;j:64;e:64;f:4;")
    a, b, c0 = operands(reg, 5)
    for level in (1, 2):
        for ps in ("0", "1"):
            check(reg, a, b, c0, level, "abc", {"STC_PRESUM_OPS": ps, "STC_ABC_DENSE": "0"})
    check(reg, a, b, c0, 2, "ab", {"STC_PRESUM_OPS": "0"})
    check(reg, a, b, c0, 1, "abc", force_slow=True)
    check(reg, a, b, c0, 2, "abc", {"STC_HOST_PIECES": "2"}, host=True)
    torch.cuda.synchronize()
    print("all cases ok")


if __name__ == "__main__":
    main()
