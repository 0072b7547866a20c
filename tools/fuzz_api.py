"""Randomised check of the public contract() API beyond tools/fuzz_gpu.py: operands in host
(numpy) or device memory, layouts that are permuted, padded (non-compact), offset and with
negative strides; the force_slow / reference_tiling / validate flags; TileConfig params; levels
0-3 (3 with allow_deep); degenerate bundles.  Each result is compared with a float64 einsum of
the same logical tensors.

Usage: python tools/fuzz_api.py [cases] [seed]      (STC_FUZZ_VERBOSE=1 prints each run first)
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


def rand_spec(rng):
    ni, nj, np_ = rng.randint(0, 3), rng.randint(0, 3), rng.randint(0, 3)
    labels = list("abcdefghijkl")
    rng.shuffle(labels)
    li, lj, lp = labels[:ni], labels[ni:ni + nj], labels[ni + nj:ni + nj + np_]
    kind = rng.random()
    ext = {}
    for l in li + lj + lp:
        if kind < 0.35:
            ext[l] = rng.choice([1, 2, 8, 16, 32, 64])
        elif kind < 0.7:
            ext[l] = rng.randint(1, 24)
        else:
            ext[l] = rng.choice([1, 3, 5, 17, 96, 130])
    size = lambda g: int(np.prod([ext[l] for l in g])) if g else 1
    while size(li) * size(lj) * size(lp) > 2 ** 25 or size(li) * size(lp) > 2 ** 22 or size(lp) * size(lj) > 2 ** 22 \
            or size(li) * size(lj) > 2 ** 22:
        l = rng.choice(li + lj + lp)
        ext[l] = max(1, ext[l] // 2)
    lc, la, lb = li + lj, li + lp, lp + lj
    for x in (lc, la, lb):
        rng.shuffle(x)
    return stc.ContractionSpec("".join(lc), "".join(la), "".join(lb), ext)


def rand_layout(rng, extents):
    """(strides, base_offset, storage size, flipped dims) of an injective layout: a random
    permutation of the dims, optional padding between them, optional negative strides."""
    nd = len(extents)
    order = list(range(nd))
    rng.shuffle(order)
    strides, run = [0] * nd, 1
    for d in order:
        strides[d] = run
        run *= extents[d]
        if rng.random() < 0.25:
            run += rng.randint(1, 5)  # padding: non-compact storage
    flips = [d for d in range(nd) if extents[d] > 1 and rng.random() < 0.15]
    base = rng.choice([0, 0, 1, 3])
    for d in flips:
        base += (extents[d] - 1) * strides[d]
        strides[d] = -strides[d]
    return tuple(strides), base, run + 3


def make(rng, nprng, extents, host):
    strides, base, size = rand_layout(rng, extents)
    data = nprng.integers(-8, 9, size).astype(np.float64) if rng.random() < 0.3 else nprng.uniform(-1, 1, size)
    # logical view for the einsum gold
    lo = base + sum(min(0, (e - 1) * s) for e, s in zip(extents, strides))
    idx = np.full(tuple(extents) if extents else (), base, dtype=np.int64)
    for d, (e, s) in enumerate(zip(extents, strides)):
        shape = [1] * len(extents)
        shape[d] = e
        idx = idx + (np.arange(e, dtype=np.int64) * s).reshape(shape)
    assert lo >= 0 and idx.max(initial=0) < size
    storage = data if host else torch.from_numpy(data).cuda()
    return stc.DenseTensor(tuple(extents), strides, storage, base), idx, data


def main(cases, seed):
    rng = random.Random(seed)
    nprng = np.random.default_rng(seed)
    worst, fails, runs, kinds = 0.0, 0, 0, {"host": 0, "device": 0}
    for case in range(cases):
        spec = rand_spec(rng)
        host = rng.random() < 0.4
        kinds["host" if host else "device"] += 1
        (a, ia, da), (b, ib, db), (c, ic, dc) = (make(rng, nprng, spec.tensor_extents(l), host)
                                                 for l in (spec.labels_a, spec.labels_b, spec.labels_c))
        ga, gb, gc = (torch.from_numpy(np.asarray(d[i]).reshape(i.shape).copy()).cuda() for d, i in ((da, ia), (db, ib), (dc, ic)))
        ref = (gc + torch.einsum(f"{spec.labels_a},{spec.labels_b}->{spec.labels_c}", ga, gb)).cpu().numpy()
        nref = float(np.linalg.norm(ref))
        for _ in range(4):
            level = rng.choice([0, 1, 1, 2, 2, 3])
            variant = rng.choice(["abc", "ab", "naive"])
            kw = {"force_slow": rng.random() < 0.15, "reference_tiling": rng.random() < 0.15,
                  "validate": rng.random() < 0.2, "allow_deep": level > 2}
            if rng.random() < 0.25 and level >= 1 and variant != "naive" and not kw["force_slow"]:
                kw["params"] = stc.TileConfig(cta_tile=rng.choice([None, (128, 128), (64, 128), (128, 64)]),
                                              stages=rng.choice([None, 2, 3, 5, 8]))
            store = dc.copy()
            cc = stc.DenseTensor(c.extents, c.strides, store if host else torch.from_numpy(store).cuda(), c.base_offset)
            if VERBOSE:
                print("RUN", case, stc.to_benchmark_line(spec), "host" if host else "dev", a.strides, a.base_offset,
                      b.strides, b.base_offset, c.strides, c.base_offset, "L", level, variant, kw, flush=True)
            try:
                st = stc.contract(spec, a, b, cc, level, variant, **kw)
            except ValueError as exc:
                if "params" in kw and "tile" in str(exc).lower():
                    continue  # a shape this problem cannot use: rejected before any device work
                raise
            runs += 1
            out = store if host else cc.data.cpu().numpy()
            err = float(np.linalg.norm(out[ic] - ref)) / max(nref, 1e-300)
            # untouched storage (padding, outside the view) must be unchanged
            mask = np.ones(out.shape, bool)
            mask[ic.reshape(-1)] = False
            clean = np.array_equal(out[mask], dc[mask])
            worst = max(worst, err)
            if not (err <= 1e-12 and clean and st.leaf_multiplies == 7 ** level):
                fails += 1
                print("FAIL", stc.to_benchmark_line(spec), "host" if host else "dev", a.strides, a.base_offset, b.strides,
                      b.base_offset, c.strides, c.base_offset, "L", level, variant, kw, "err", err, "clean", clean, flush=True)
    print(f"{cases} cases, {runs} runs ({kinds}): {fails} failures, worst rel err {worst:.3e}", flush=True)
    return fails


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    s = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    sys.exit(1 if main(n, s) else 0)
