"""Randomised GPU check: random contractions (labels, extents, permuted layouts, storage
offsets) through every variant and level, against a classical torch.einsum in FP64.

Sizes are drawn so that many cases hit the box-regular fused path (extents that are
multiples of 16) and many hit the repacked / gather paths.  Prints failures and a summary.

Usage: python tools/fuzz_gpu.py [cases] [seed]
"""

import os
import pathlib
import random
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_1704_03092_b200 as stc  # noqa: E402


VERBOSE = bool(os.environ.get("STC_FUZZ_VERBOSE"))


def rand_case(rng):
    ni, nj, np_ = rng.randint(1, 3), rng.randint(1, 3), rng.randint(1, 3)
    labels = list("abcdefghijkl")
    rng.shuffle(labels)
    li, lj, lp = labels[:ni], labels[ni:ni + nj], labels[ni + nj:ni + nj + np_]
    regular = rng.random() < 0.6
    ext = {}
    for l in li + lj + lp:
        ext[l] = rng.choice([32, 64, 128]) if regular else rng.randint(1, 40)
    if regular:  # bundles large enough for 128-wide tiles of 2^L quadrants: the direct TMA path
        for group in (li, lj, lp):
            while np.prod([ext[l] for l in group]) < 512:
                ext[rng.choice(group)] *= 2
        if rng.random() < 0.3:  # an I or J bundle of 256: 64-wide quadrants at L2 (64 x 256 / 256 x 64 tiles)
            group = li if rng.random() < 0.5 else lj
            for l in group:
                ext[l] = 1
            ext[group[0]] = 256 if len(group) == 1 else 16
            if len(group) > 1:
                ext[group[1]] = 16
    # keep the problem moderate
    while np.prod([ext[l] for l in li]) * np.prod([ext[l] for l in lj]) * np.prod([ext[l] for l in lp]) > 2 ** 28:
        l = rng.choice(li + lj + lp)
        ext[l] = max(1, ext[l] // 2)
    lc, la, lb = li + lj, li + lp, lp + lj
    for x in (lc, la, lb):
        rng.shuffle(x)
    return stc.ContractionSpec("".join(lc), "".join(la), "".join(lb), ext)


def tensor(spec, labels, gen, offset):
    e = spec.tensor_extents(labels)
    n = int(np.prod(e))
    flat = torch.rand(n + offset, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
    return torch.as_strided(flat, e, tuple(int(np.prod(e[i + 1:])) for i in range(len(e))), offset)


def main(cases, seed):
    rng = random.Random(seed)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    worst, fails, paths = 0.0, 0, {"fast": 0, "slow": 0}
    for case in range(cases):
        spec = rand_case(rng)
        off = rng.choice([0, 0, 1, 2])
        a, b, c = (tensor(spec, spec.labels_a, gen, off), tensor(spec, spec.labels_b, gen, off),
                   tensor(spec, spec.labels_c, gen, 0))
        ref = c + torch.einsum(f"{spec.labels_a},{spec.labels_b}->{spec.labels_c}", a, b)
        nref = torch.linalg.vector_norm(ref).item()
        for level, variant, env in [(lv, var, env) for lv in (0, 1, 2) for var in ("abc", "ab", "naive")
                                    for env in ({}, {"STC_PRESUM_OPS": "1"}, {"STC_PRESUM_OPS": "0"})
                                    if not (env and (lv == 0 or var == "naive"))]:
                os.environ.pop("STC_PRESUM_OPS", None)
                os.environ.update(env)
                cc = c.clone()
                if VERBOSE:  # the case about to run (a crash is then attributable)
                    print("RUN", case, stc.to_benchmark_line(spec), "offset", off, "L", level, variant, env, flush=True)
                st = stc.contract(spec, a, b, cc, level, variant)
                if VERBOSE:
                    torch.cuda.synchronize()
                paths["fast" if st.fast_blocks else "slow"] += 1
                err = torch.linalg.vector_norm(cc - ref).item() / max(nref, 1e-300)
                worst = max(worst, err)
                if not err <= 1e-12:
                    fails += 1
                    print("FAIL", stc.to_benchmark_line(spec), "offset", off, "L", level, variant, env, err, flush=True)
    os.environ.pop("STC_PRESUM_OPS", None)
    print(f"{cases} cases x 13 runs: {fails} failures, worst rel err {worst:.3e}, staging {paths}", flush=True)
    return fails


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    s = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    sys.exit(1 if main(n, s) else 0)
