"""GPU tests of the kernel-level API and of full-size BASELINE configs.

Reference test models: pkg/tests/test_scatter.py (views), test_driver.py (fused
term, dense GEMM), test_kernels.py (accumulate / unpack), test_strassen.py and
test_acceptance.py (integer exactness, variants agree, determinism).
"""

import numpy as np
import pytest

import golden_io
import oracle
import paper_1704_03092_b200 as stc
from paper_1704_03092_b200 import shard

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _rm(e):
    return tuple(int(np.prod(e[i + 1:])) for i in range(len(e)))


def _tensors(spec, seed, fill="random", device=None):
    def t(labels, s, zero=False):
        e = spec.tensor_extents(labels)
        n = int(np.prod(e))
        rng = np.random.default_rng(s)
        if zero:
            data = np.zeros(n)
        elif fill == "int":
            data = rng.integers(-1024, 1025, n).astype(np.float64)
        else:
            data = rng.uniform(-1, 1, n)
        x = stc.DenseTensor(e, _rm(e), data)
        return x.to_device() if device else x
    return t(spec.labels_a, seed), t(spec.labels_b, seed + 1), t(spec.labels_c, seed + 2, zero=True)


# ---- subsystem (1): device-built views bitwise against the reference -------------
def test_device_views_match_reference_golden():
    import torch

    meta, arr = golden_io.view_cases()
    for k, cs in enumerate(meta):
        span = cs["base"] + sum((e - 1) * s for e, s in zip(cs["ext"], cs["strides"])) + 1
        t = stc.DenseTensor(cs["ext"], cs["strides"], torch.zeros(max(span, int(np.prod(cs["ext"]))),
                                                                   dtype=torch.float64, device="cuda"), cs["base"])
        axes = {lab: i for i, lab in enumerate(cs["labels"])}
        v = stc.make_view(t, cs["rows"], cs["cols"], axes, cs["rb"], cs["cb"])
        views = {0: v} if cs["level"] == 0 else stc.quadrant_views(v, cs["level"])
        assert len(views) == cs["nquads"]
        for q, qv in views.items():
            for name in ("rscat", "cscat", "rbs", "cbs"):
                assert np.array_equal(getattr(qv, name).cpu().numpy(), arr[f"c{k}_q{q}_{name}"]), (k, q, name)


def test_view_get_set_pad_semantics():
    import torch

    t = stc.DenseTensor((3, 2), (1, 3), torch.zeros(6, dtype=torch.float64, device="cuda"))
    p = stc.pad_view(stc.matrix_view(t, 2, 2), 4, 2)
    assert p.rscat.tolist()[-1] == stc.PAD and p.rbs.tolist() == [1, 0]
    p.set(3, 0, 5.0)  # dropped
    assert not t.data.any().item()
    assert p.get(3, 0) == 0.0


# ---- subsystems (2)+(3): one fused term -----------------------------------------
def test_fused_strassen_term_m0_integers_exact():
    import torch

    rng = np.random.default_rng(11)
    a = rng.integers(-9, 10, (4, 4)).astype(float)
    b = rng.integers(-9, 10, (4, 4)).astype(float)
    c = rng.integers(-9, 10, (4, 4)).astype(float)
    expect = c.copy()
    m0 = (a[:2, :2] + a[2:, 2:]) @ (b[:2, :2] + b[2:, 2:])
    expect[:2, :2] += m0
    expect[2:, 2:] += m0

    def dev(x):  # column-major device DenseTensor
        return stc.DenseTensor((4, 4), (1, 4), torch.from_numpy(x.ravel(order="F").copy()).cuda())

    ta, tb, tc = dev(a), dev(b), dev(c)
    va, vb, vc = stc.matrix_view(ta, 2, 2), stc.matrix_view(tb, 2, 2), stc.matrix_view(tc, 2, 2)
    q = lambda v, r, s: stc.split_view(v, r, s)
    prim = stc.FusedPrimitive(
        stc.OperandTermSide([q(va, (0, 2), (0, 2)), q(va, (2, 4), (2, 4))], [1, 1]),
        stc.OperandTermSide([q(vb, (0, 2), (0, 2)), q(vb, (2, 4), (2, 4))], [1, 1]),
        stc.OperandTermSide([q(vc, (0, 2), (0, 2)), q(vc, (2, 4), (2, 4))], [1, 1]),
    )
    st = stc.run_fused(prim, validate=True)
    assert st.leaf_multiplies == 1
    assert np.array_equal(tc.data.cpu().numpy().reshape(4, 4, order="F"), expect)


def test_validate_rejects_overlapping_targets():
    import torch

    tc = stc.DenseTensor((4, 4), (1, 4), torch.zeros(16, dtype=torch.float64, device="cuda"))
    vc = stc.matrix_view(tc, 2, 2)
    ta = stc.DenseTensor((2, 2), (1, 2), torch.zeros(4, dtype=torch.float64, device="cuda"))
    side = stc.OperandTermSide([stc.matrix_view(ta, 2, 2)], [1])
    prim = stc.FusedPrimitive(side, stc.OperandTermSide([stc.matrix_view(ta, 2, 2)], [1]),
                              stc.OperandTermSide([stc.split_view(vc, (0, 2), (0, 2)),
                                                   stc.split_view(vc, (0, 2), (1, 3))], [1, 1]))
    with pytest.raises(ValueError, match="overlap"):
        stc.run_fused(prim, validate=True)


def test_run_gemm_dense_and_errors():
    import torch

    rng = np.random.default_rng(3)
    a, b, c = rng.uniform(-1, 1, (130, 70)), rng.uniform(-1, 1, (70, 150)), rng.uniform(-1, 1, (130, 150))
    cm = lambda x: torch.from_numpy(np.asfortranarray(x)).cuda()
    tc = cm(c)
    stc.run_gemm_dense(tc, cm(a), cm(b))
    ref = c + a @ b
    assert np.linalg.norm(tc.cpu().numpy() - ref) / np.linalg.norm(ref) < 1e-13
    with pytest.raises(ValueError, match="column-major"):
        stc.run_gemm_dense(cm(c), torch.from_numpy(a).cuda(), cm(b))
    with pytest.raises(ValueError, match="shape"):
        stc.run_gemm_dense(cm(c), cm(a), cm(b[:60]))


# ---- subsystem (4): accumulate / unpack ------------------------------------------
def test_accumulate_and_unpack_match_element_semantics():
    import torch

    spec = stc.parse_benchmark_line("abc dca db & a:4;b:12;c:2;d:8;")
    c = stc.make_dense_tensor(spec.tensor_extents(spec.labels_c), "random", 6, device="cuda")
    axes = {lab: i for i, lab in enumerate(spec.labels_c)}
    view = stc.make_view(c, spec.bundle_i, spec.bundle_j, axes, 8, 4)
    before = view.to_dense().cpu().numpy()
    mat = np.random.default_rng(7).uniform(-1, 1, (8, 12))
    st = stc.RunStats()
    stc.accumulate_dense_to_view(mat, -1, view, st)
    assert np.array_equal(view.to_dense().cpu().numpy(), before - mat)
    with pytest.raises(ValueError, match="shape"):
        stc.accumulate_dense_to_view(np.zeros((12, 8)), 1, view, st)
    # unpack: cancelling views give zeros; quadrant sum equals the element oracle
    t = stc.make_dense_tensor((8, 2, 4), "sequence", device="cuda")
    v = stc.make_view(t, "ac", "d", {"d": 0, "c": 1, "a": 2}, 4, 4)
    assert not stc.unpack_to_dense(stc.OperandTermSide([v, v], [1, -1])).any().item()
    top, bottom = stc.split_view(v, (0, 4), (0, 4)), stc.split_view(v, (4, 8), (4, 8))
    out = stc.unpack_to_dense(stc.OperandTermSide([top, bottom], [1, 1]))
    assert np.array_equal(out.cpu().numpy(), top.to_dense().cpu().numpy() + bottom.to_dense().cpu().numpy())


def test_device_relative_error_matches_oracle():
    a = stc.make_dense_tensor((6, 5, 4), "random", 1)
    r = stc.make_dense_tensor((6, 5, 4), "random", 2)
    dev = stc.relative_error(a.to_device(), r.to_device())
    assert dev == pytest.approx(oracle.relative_error(a, r), rel=1e-13)
    z = stc.make_dense_tensor((2, 2), device="cuda")
    assert stc.relative_error(z, z) == 0.0
    import math
    assert stc.relative_error(stc.make_dense_tensor((2, 2), "sequence", device="cuda"), z) == math.inf


# ---- larger problems: integers exact, tickets, PAD, multiple tiles ----------------
@pytest.mark.parametrize("level", [1, 2])
def test_integer_exact_multi_tile_with_pad(level):
    spec = stc.parse_benchmark_line("abc dca db & a:37;b:150;c:9;d:170;")
    a, b, c0 = _tensors(spec, 9, fill="int")
    ref = c0.copy()
    oracle.contract_reference(spec, a, b, ref, threads=8)
    for variant in stc.Variant:
        for kw in ({}, {"force_slow": True}, {"reference_tiling": True}):
            c = c0.copy()
            stc.contract(spec, a, b, c, level, variant, **kw)
            assert np.array_equal(c.data, ref.data), (variant, kw)


def test_bitwise_determinism_with_tickets():
    """L2 ABC with many tiles per term: C-tile updates serialised by tickets."""
    spec = stc.parse_benchmark_line("abij abef efij & a:32;b:32;i:32;j:32;e:32;f:32;")
    a, b, c0 = _tensors(spec, 21, device=True)
    outs = []
    for _ in range(3):
        c = c0.copy()
        stc.contract(spec, a, b, c, 2, "abc")
        outs.append(c.data.cpu().numpy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def _sampled_exact(spec, a, b, c, nsamples=256, seed=0):
    """max relative deviation of sampled C entries from fp64 dot products on the host."""
    A, B, C = a.to_host(), b.to_host(), c.to_host()
    rng = np.random.default_rng(seed)
    def bundle_offsets(bundle, labels, t):
        offs = np.zeros(1, np.int64)
        for lab in bundle:
            ax = labels.index(lab)
            offs = (offs[:, None] + np.arange(t.extents[ax], dtype=np.int64)[None, :] * t.strides[ax]).ravel(order="F")
        return offs
    ai = bundle_offsets(spec.bundle_i, spec.labels_a, A) + A.base_offset
    ap = bundle_offsets(spec.bundle_p, spec.labels_a, A)
    bp = bundle_offsets(spec.bundle_p, spec.labels_b, B) + B.base_offset
    bj = bundle_offsets(spec.bundle_j, spec.labels_b, B)
    ci = bundle_offsets(spec.bundle_i, spec.labels_c, C) + C.base_offset
    cj = bundle_offsets(spec.bundle_j, spec.labels_c, C)
    worst = 0.0
    for _ in range(nsamples):
        i, j = rng.integers(len(ai)), rng.integers(len(bj))
        exact = float(np.dot(A.data[ai[i] + ap], B.data[bp + bj[j]]))
        got = float(C.data[ci[i] + cj[j]])
        worst = max(worst, abs(got - exact) / max(1.0, abs(exact)))
    return worst


@pytest.mark.parametrize("line", ["aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;",          # cfg2
                                  "abcij eafbc ifje & a:50;b:7;c:13;i:70;j:45;e:90;f:33;"])  # cfg4
def test_full_size_configs_against_classical_gpu_and_samples(line):
    spec = stc.parse_benchmark_line(line)
    a, b, c0 = _tensors(spec, 13, device=True)
    ref = c0.copy()
    stc.contract(spec, a, b, ref, 0, "abc")
    assert _sampled_exact(spec, a, b, ref) < 1e-12
    runs = [(2, "abc"), (2, "ab"), (2, "naive"), (1, "abc")] if "aibj" in line else \
        [(1, "ab"), (1, "naive"), (2, "ab"), (2, "naive"), (2, "abc")]
    for level, variant in runs:
        c = c0.copy()
        stc.contract(spec, a, b, c, level, variant)
        assert stc.relative_error(c, ref) < 1e-12, (level, variant)


def test_sharded_path_on_one_gpu_matches_unsharded():
    """n-split (subsystem 5): ranks run one after another on this GPU, no collective."""
    spec = stc.parse_benchmark_line("abcijk abcefg efgijk & a:8;b:8;c:8;i:8;j:8;k:8;e:8;f:8;g:8;")
    a, b, c0 = _tensors(spec, 17, device=True)
    full = c0.copy()
    stc.contract(spec, a, b, full, 2, "abc")
    c = c0.copy()
    for rank in range(4):
        shard.contract_sharded(spec, a, b, c, 2, "abc", rank, 4)
    assert stc.relative_error(c, full) < 1e-12


def test_grid_blocks_on_one_gpu_match_unsharded():
    """2-D split: the 2 x 2 grid's blocks run one after another on
    this GPU; every C element is owned by one block, no reduction."""
    spec = stc.parse_benchmark_line("abcijk abcefg efgijk & a:8;b:8;c:8;i:8;j:8;k:8;e:8;f:8;g:8;")
    a, b, c0 = _tensors(spec, 19, device=True)
    full = c0.copy()
    stc.contract(spec, a, b, full, 2, "abc")
    for gm, gn in ((2, 2), (4, 1), (1, 2)):
        c = c0.copy()
        for rank in range(gm * gn):
            shard.contract_grid(spec, a, b, c, 2, "abc", rank, gm, gn)
        assert stc.relative_error(c, full) < 1e-12, (gm, gn)


# ---- small-problem path: CUDA-graph replay of a plan's launch sequence ------------
def test_graph_replay_follows_inputs_and_pointers():
    # a small problem replays a graph captured for its (A, B, C, workspace) pointers: new
    # values in the same buffers, a second C buffer (a second graph) and the graph-free
    # path must all give the oracle's result, bitwise equal to one another
    import os

    import torch

    spec = stc.parse_benchmark_line("abij abef efij & a:24;b:24;i:24;j:24;e:24;f:24;")  # cfg1
    a, b, c = _tensors(spec, 1301, fill="int")
    da, db = a.to_device(), b.to_device()
    cs = [c.to_device(), c.to_device()]
    for level, variant in ((1, "abc"), (2, "abc"), (1, "ab"), (2, "naive")):
        for it in range(4):
            # integer values: the result is exact, so every path must equal the oracle
            vals = np.random.default_rng(it + 10 * level).integers(-64, 65, da.data.numel()).astype(np.float64)
            da.data.copy_(torch.from_numpy(vals))
            ha = stc.DenseTensor(a.extents, a.strides, vals)
            cd = cs[it % 2]
            cd.data.zero_()
            st = stc.contract(spec, da, db, cd, level, variant)
            ref = stc.DenseTensor(c.extents, c.strides, np.zeros(c.data.size))
            oracle.contract_reference(spec, ha, b, ref)
            assert np.array_equal(cd.to_host().data, ref.data), (level, variant, it)
            assert st.leaf_multiplies == 7 ** level
        os.environ["STC_NO_GRAPH"] = "1"  # the direct launches, same inputs as the last replay
        try:
            cs[0].data.zero_()
            stc.contract(spec, da, db, cs[0], level, variant)
        finally:
            del os.environ["STC_NO_GRAPH"]
        assert np.array_equal(cs[0].to_host().data, ref.data), (level, variant)


# ---- degenerate specs the reference accepts (empty bundles, rank-0 C, extent-1 labels) -------
DEGENERATE = [
    ("ij", "i", "j", {"i": 4, "j": 5}),                      # empty P bundle: outer product (k = 1)
    ("i", "ie", "e", {"i": 4, "e": 5}),                      # empty J bundle: matrix-vector (n = 1)
    ("j", "e", "ej", {"j": 4, "e": 5}),                      # empty I bundle (m = 1)
    ("", "e", "e", {"e": 37}),                               # rank-0 C: dot product
    ("ij", "ie", "ej", {"i": 1, "j": 1, "e": 1}),            # all extents 1 (quadrants are PAD)
    ("abij", "aeb", "ije", {"a": 1, "b": 300, "i": 1, "j": 3, "e": 130}),  # extent-1 labels inside bundles
    ("ij", "i", "j", {"i": 300, "j": 200}),                  # outer product over several tiles
]


@pytest.mark.parametrize("case", DEGENERATE, ids=lambda c: f"{c[0] or '0'}-{c[1]}-{c[2]}")
@pytest.mark.parametrize("where", ["device", "host"])
def test_degenerate_specs_match_oracle_exactly(case, where):
    """Integer data, so every level and variant must equal the classical oracle exactly;
    the reference runs all of these (7^L leaves on PAD-only quadrants included)."""
    lc, la, lb, ext = case
    spec = stc.ContractionSpec(lc, la, lb, ext)
    a, b, c0 = _tensors(spec, 3, fill="int")
    c0.data[:] = np.random.default_rng(9).integers(-50, 51, c0.data.size).astype(np.float64)
    gold = c0.copy()
    oracle.contract_reference(spec, a, b, gold)
    for level in (0, 1, 2):
        for variant in ("abc", "ab", "naive"):
            if where == "device":
                ad, bd, c = a.to_device(), b.to_device(), c0.to_device()
                st = stc.contract(spec, ad, bd, c, level, variant)
                got = c.to_host().data
            else:
                c = c0.copy()
                st = stc.contract(spec, a, b, c, level, variant)
                got = c.data
            assert st.leaf_multiplies == 7 ** level
            assert np.array_equal(got, gold.data), (case, where, level, variant)
