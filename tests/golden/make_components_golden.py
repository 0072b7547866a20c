"""Golden vectors of the reference's component calls (pack_a, pack_b, microkernel).

Run in the build container only (imports the read-only reference checkout):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_components_golden.py

Writes tests/golden/components.npz + components.json: seeded parents, the views'
scatter vectors, and the REFERENCE's packed panels / updated targets with its
fast / slow counts (kernels.py:166-233).  Tests read only the committed files.

Cases: dense and permuted parents, Strassen quadrant sides with +/-1 coefficients
(1-4 views, odd sizes so some quadrants carry PAD), fringe blocks, both store
paths (force_slow), k = 0 / 1 / odd depths, repeated (identical) targets.
"""

from __future__ import annotations

import json
import pathlib
import sys

import numpy as np

REF = pathlib.Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

import strassen_tc as st  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent


def parent(rng, m, n, order, integer=False):
    """An m x n parent matrix as a 2-axis DenseTensor, column- or row-major, with a base offset."""
    base = int(rng.integers(0, 5))
    strides = (1, m) if order == "F" else (n, 1)
    size = base + m * n
    data = rng.integers(-4, 5, size).astype(np.float64) if integer else rng.uniform(-1, 1, size)
    return st.DenseTensor((m, n), strides, data, base)


def side_of(t, rb, cb, level, ops):
    v = st.matrix_view(t, rb, cb)
    if level == 0:
        views = [v] * len(ops)
    else:
        q = st.quadrant_views(v, level)
        views = [q[i] for i, _ in ops]
    return st.OperandTermSide(views, [c for _, c in ops])


def main():
    rng = np.random.default_rng(170403092)
    arrays, meta = {}, {"pack": [], "micro": []}
    P = st.BlockingParams(mc=16, nc=16, kc=8, mr=8, nr=4, kr=4)
    # ---- pack_a / pack_b
    pack_cases = [
        # (which, m, n, order, level, ops, x block, k block, force_slow)
        (0, 16, 8, "F", 0, [(0, 1)], (0, 16), (0, 8), False),
        (0, 16, 8, "C", 0, [(0, -1)], (8, 16), (4, 8), False),
        (0, 16, 8, "F", 0, [(0, 1), (0, -1)], (0, 16), (0, 8), False),
        (0, 32, 16, "F", 1, [(0, 1), (3, 1)], (0, 16), (0, 8), False),
        (0, 32, 16, "C", 1, [(1, 1), (3, -1)], (8, 16), (4, 8), True),
        (0, 27, 13, "F", 1, [(2, -1), (3, 1)], (8, 14), (4, 7), False),    # PAD quadrants, fringes
        (0, 27, 13, "F", 2, [(5, 1), (15, -1), (10, 1)], (0, 7), (0, 4), False),
        (0, 45, 30, "C", 2, [(0, 1), (5, 1), (10, -1), (15, 1)], (8, 12), (0, 8), False),
        (1, 8, 16, "F", 0, [(0, 1)], (0, 16), (0, 8), False),
        (1, 8, 16, "C", 0, [(0, 1), (0, 1)], (4, 12), (4, 8), False),
        (1, 16, 32, "C", 1, [(0, 1), (2, -1)], (0, 16), (0, 8), False),
        (1, 13, 27, "F", 1, [(1, 1), (3, 1)], (4, 14), (4, 7), True),
        (1, 13, 27, "C", 2, [(7, -1), (13, 1)], (0, 7), (0, 4), False),
        (1, 30, 45, "F", 2, [(3, 1), (6, -1), (9, 1), (12, -1)], (8, 12), (0, 8), False),
    ]
    for idx, (which, m, n, order, level, ops, xb, kb, slow) in enumerate(pack_cases):
        t = parent(rng, m, n, order, integer=idx % 5 == 4)
        rb, cb = (P.mr, P.kr) if which == 0 else (P.kr, P.nr)
        side = side_of(t, rb, cb, level, ops)
        stats = st.RunStats()
        if which == 0:
            buf = st.PackedBuffer.a_panel(P, xb[1] - xb[0], kb[1] - kb[0])
            st.pack_a(side, xb, kb, P, buf, stats, force_slow=slow)
        else:
            buf = st.PackedBuffer.b_panel(P, xb[1] - xb[0], kb[1] - kb[0])
            st.pack_b(side, kb, xb, P, buf, stats, force_slow=slow)
        key = f"pack{idx}"
        arrays[key + "_data"] = t.data
        arrays[key + "_out"] = buf.data
        for v_i, v in enumerate(side.views):
            arrays[f"{key}_r{v_i}"] = v.rscat
            arrays[f"{key}_c{v_i}"] = v.cscat
        meta["pack"].append(dict(which=which, rb=rb, cb=cb, nviews=len(side.views), coeffs=list(side.coeffs),
                                 x=list(xb), k=list(kb), force_slow=slow, fast=stats.fast_blocks,
                                 slow=stats.slow_blocks, row_unit=side.views[0].row_unit_stride,
                                 col_unit=side.views[0].col_unit_stride, shape=[m, n], level=level))
    # ---- microkernel
    micro_cases = [
        # (mr, nr, k, avail, m, n, order, level, targets [(quadrant, i0, j0, coeff)], force_slow)
        (8, 4, 8, 8, 16, 8, "F", 0, [(0, 0, 0, 1)], False),
        (8, 4, 5, 8, 16, 8, "C", 0, [(0, 8, 4, -1)], False),
        (8, 4, 1, 3, 16, 8, "F", 0, [(0, 8, 0, 1), (0, 8, 0, 1)], False),       # identical targets, in order
        (8, 4, 0, 4, 16, 8, "F", 0, [(0, 0, 0, 1)], False),                     # k = 0: untouched
        (8, 4, 7, 7, 32, 16, "F", 1, [(0, 0, 0, 1), (3, 0, 0, -1)], False),
        (8, 4, 8, 8, 32, 16, "C", 1, [(1, 8, 4, 1), (2, 8, 4, 1)], True),
        (8, 4, 6, 8, 27, 13, "F", 1, [(1, 8, 4, -1), (3, 8, 4, 1)], False),     # fringe + PAD dropped
        (8, 4, 8, 8, 45, 30, "C", 2, [(0, 8, 4, 1), (5, 8, 4, -1), (10, 8, 4, 1), (15, 8, 4, 1)], False),
        (4, 4, 9, 9, 18, 18, "F", 1, [(0, 4, 8, 1), (3, 8, 8, -1)], False),
    ]
    for idx, (mr, nr, k, avail, m, n, order, level, tg, slow) in enumerate(micro_cases):
        t = parent(rng, m, n, order, integer=idx % 4 == 3)
        v = st.matrix_view(t, mr, nr)
        quads = {0: v} if level == 0 else st.quadrant_views(v, level)
        a = rng.uniform(-1, 1, (mr, avail))
        b = rng.uniform(-1, 1, (avail, nr))
        key = f"micro{idx}"
        arrays[key + "_a"], arrays[key + "_b"], arrays[key + "_before"] = a, b, t.data.copy()
        stats = st.RunStats()
        st.microkernel(a, b, k, [(quads[q], i0, j0, co) for q, i0, j0, co in tg], stats, force_slow=slow)
        arrays[key + "_after"] = t.data
        for g, (q, _, _, _) in enumerate(tg):
            arrays[f"{key}_r{g}"] = quads[q].rscat
            arrays[f"{key}_c{g}"] = quads[q].cscat
        meta["micro"].append(dict(mr=mr, nr=nr, k=k, targets=[[i0, j0, co] for _, i0, j0, co in tg],
                                  force_slow=slow, fast=stats.fast_updates, slow=stats.slow_updates,
                                  row_unit=v.row_unit_stride, col_unit=v.col_unit_stride))
    np.savez_compressed(OUT / "components.npz", **arrays)
    (OUT / "components.json").write_text(json.dumps(meta, indent=1))
    print(f"{len(meta['pack'])} pack cases, {len(meta['micro'])} microkernel cases")


if __name__ == "__main__":
    main()
