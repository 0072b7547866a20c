"""GPU: the reference's component API (PackedBuffer, pack_a, pack_b, microkernel,
contract_reference) on the device.

Bitwise against the REFERENCE's own outputs (tests/golden/components.npz), bitwise against
the CPU oracle on larger seeded cases, and the reference's unit-test properties
(pkg/tests/test_kernels.py:67-268: cancelling views, linearity, path equivalence, PAD
neutrality, validation, k = 0, negative coefficient, PAD writes dropped)."""

import numpy as np
import pytest

import oracle
import paper_1704_03092_b200 as stc
from test_oracle_components import load

pytestmark = pytest.mark.gpu
P = stc.BlockingParams(mc=16, nc=16, kc=8, mr=8, nr=4, kr=4)


def bits(x):
    x = x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)
    return np.ascontiguousarray(x, dtype=np.float64).view(np.int64)


def parent(data):
    import torch

    d = torch.from_numpy(np.ascontiguousarray(data, dtype=np.float64)).cuda()
    return stc.DenseTensor((d.numel(),), (1,), d)


def view(base, rscat, cscat, rb, cb, ru=1, cu=1):
    return stc.BlockScatterView.from_scatter(base, rscat, cscat, rb, cb, ru, cu)


def test_pack_matches_reference_golden_bitwise():
    meta, arr = load()
    for k, cs in enumerate(meta["pack"]):
        key = f"pack{k}"
        base = parent(arr[key + "_data"])
        side = stc.OperandTermSide([view(base, arr[f"{key}_r{t}"], arr[f"{key}_c{t}"], cs["rb"], cs["cb"],
                                         cs["row_unit"], cs["col_unit"]) for t in range(cs["nviews"])], cs["coeffs"])
        x, kk = cs["x"], cs["k"]
        stats = stc.RunStats()
        if cs["which"] == 0:
            buf = stc.PackedBuffer.a_panel(P, x[1] - x[0], kk[1] - kk[0])
            stc.pack_a(side, x, kk, P, buf, stats, force_slow=cs["force_slow"])
        else:
            buf = stc.PackedBuffer.b_panel(P, x[1] - x[0], kk[1] - kk[0])
            stc.pack_b(side, kk, x, P, buf, stats, force_slow=cs["force_slow"])
        want = arr[key + "_out"]
        assert tuple(buf.data.shape) == want.shape, (k, buf.data.shape, want.shape)
        assert np.array_equal(bits(buf.data), bits(want)), k
        assert (stats.fast_blocks, stats.slow_blocks) == (cs["fast"], cs["slow"]), k


def test_microkernel_matches_reference_golden_bitwise():
    meta, arr = load()
    for k, cs in enumerate(meta["micro"]):
        key = f"micro{k}"
        base = parent(arr[key + "_before"])
        tg = [(view(base, arr[f"{key}_r{g}"], arr[f"{key}_c{g}"], cs["mr"], cs["nr"], cs["row_unit"], cs["col_unit"]),
               i0, j0, co) for g, (i0, j0, co) in enumerate(cs["targets"])]
        stats = stc.RunStats()
        stc.microkernel(arr[key + "_a"], arr[key + "_b"], cs["k"], tg, stats, force_slow=cs["force_slow"])
        assert np.array_equal(bits(base.data), bits(arr[key + "_after"])), k
        assert (stats.fast_updates, stats.slow_updates) == (cs["fast"], cs["slow"]), k


@pytest.mark.parametrize("which", [0, 1])
def test_pack_quadrant_sides_match_oracle_bitwise(which):
    """Level-2 quadrant sides of a permuted rank-4 tensor (PAD quadrants), 96 x 64 blocks."""
    import torch

    rng = np.random.default_rng(11 + which)
    big = stc.BlockingParams(mc=96, nc=96, kc=64, mr=8, nr=4, kr=4)
    ext, perm = (32, 3, 16, 5), (2, 0, 3, 1)          # rows: axes 0, 1 (96); cols: axes 2, 3 (80)
    order = np.argsort(perm)
    strides = [0] * 4
    run = 1
    for ax in order:
        strides[ax] = run
        run *= ext[ax]
    t = stc.DenseTensor(ext, tuple(strides), torch.from_numpy(rng.uniform(-1, 1, run)).cuda(), 0)
    rb, cb = (big.mr, big.kr) if which == 0 else (big.kr, big.nr)
    v = stc.make_view(t, "ab", "cd", {"a": 0, "b": 1, "c": 2, "d": 3}, rb, cb)
    q = stc.quadrant_views(v, 2)
    ids, coeffs = [0, 5, 10, 15], [1, -1, 1, 1]
    side = stc.OperandTermSide([q[i] for i in ids], coeffs)
    xlim, klim = (side.m, side.n) if which == 0 else (side.n, side.m)
    xb, kb = (8 if which == 0 else 4, xlim), (4, klim)
    stats = stc.RunStats()
    if which == 0:
        buf = stc.PackedBuffer.a_panel(big, xb[1] - xb[0], kb[1] - kb[0])
        stc.pack_a(side, xb, kb, big, buf, stats)
    else:
        buf = stc.PackedBuffer.b_panel(big, xb[1] - xb[0], kb[1] - kb[0])
        stc.pack_b(side, kb, xb, big, buf, stats)
    want, fast, slow = oracle.pack_panel(which, t.data.cpu().numpy(), [q[i].rscat.cpu().numpy() for i in ids],
                                         [q[i].cscat.cpu().numpy() for i in ids], rb, cb, coeffs, xb, kb,
                                         row_unit=q[0].row_unit_stride, col_unit=q[0].col_unit_stride)
    assert np.array_equal(bits(buf.data), bits(want))
    assert (stats.fast_blocks, stats.slow_blocks) == (fast, slow) and fast + slow > 0


def _dense_side(m, n, seed, rb, cb, coeffs=(1,)):
    import torch

    t = stc.DenseTensor((m, n), (1, m), torch.from_numpy(np.random.default_rng(seed).uniform(-1, 1, m * n)).cuda())
    return t, stc.OperandTermSide([stc.matrix_view(t, rb, cb)] * len(coeffs), coeffs)


def test_packed_buffer_layout():
    buf = stc.PackedBuffer.a_panel(P)
    assert tuple(buf.data.shape) == (2, 8, 8) and buf.data.is_contiguous() and buf.data.data_ptr() % 64 == 0
    assert tuple(stc.PackedBuffer.b_panel(P).data.shape) == (4, 8, 4)
    assert buf.n_slivers == 2 and buf.element(1, 2, 3) == 0.0


def test_pack_cancelling_views_and_linearity():
    import torch

    t, side = _dense_side(8, 8, 3, 8, 4, (1, -1))
    buf = stc.PackedBuffer.a_panel(P, 8, 8)
    buf.data.fill_(7.0)
    stc.pack_a(side, (0, 8), (0, 8), P, buf, stc.RunStats())
    assert not buf.data.any().item()
    # two equal views: exactly twice the single view (bitwise: x + x is exact)
    _, two = _dense_side(8, 16, 4, 4, 4, (1, 1))
    one = stc.OperandTermSide(two.views[:1], [1])
    b1, b2 = stc.PackedBuffer.b_panel(P, 16, 8), stc.PackedBuffer.b_panel(P, 16, 8)
    stc.pack_b(one, (0, 8), (0, 16), P, b1, stc.RunStats())
    stc.pack_b(two, (0, 8), (0, 16), P, b2, stc.RunStats())
    assert torch.equal(b2.data, 2 * b1.data)


def test_pack_path_equivalence_and_pad_neutrality():
    import torch

    t, side = _dense_side(16, 8, 5, 8, 4)
    fast, slow = stc.PackedBuffer.a_panel(P, 16, 8), stc.PackedBuffer.a_panel(P, 16, 8)
    s1, s2 = stc.RunStats(), stc.RunStats()
    stc.pack_a(side, (0, 16), (0, 8), P, fast, s1)
    stc.pack_a(side, (0, 16), (0, 8), P, slow, s2, force_slow=True)
    assert torch.equal(fast.data, slow.data)
    assert (s1.fast_blocks, s1.slow_blocks, s2.fast_blocks, s2.slow_blocks) == (4, 0, 0, 4)
    # a padded view packs to the unpadded panel plus zeros
    padded = stc.OperandTermSide([stc.pad_view(side.views[0], 24, 8)], [1])
    big = stc.PackedBuffer.a_panel(stc.BlockingParams(mc=24, nc=16, kc=8, mr=8, nr=4, kr=4), 24, 8)
    stc.pack_a(padded, (0, 24), (0, 8), stc.BlockingParams(mc=24, nc=16, kc=8, mr=8, nr=4, kr=4), big, stc.RunStats())
    assert torch.equal(big.data[:2], fast.data) and not big.data[2].any().item()


def test_pack_geometry_validation():
    t, side = _dense_side(16, 8, 6, 8, 4)
    buf = stc.PackedBuffer.a_panel(P, 16, 8)
    with pytest.raises(ValueError, match="geometry"):
        stc.pack_b(side, (0, 8), (0, 8), P, stc.PackedBuffer.b_panel(P), stc.RunStats())
    with pytest.raises(ValueError, match="out of bounds"):
        stc.pack_a(side, (0, 24), (0, 8), P, buf, stc.RunStats())
    with pytest.raises(ValueError, match="multiple of"):
        stc.pack_a(side, (4, 12), (0, 8), P, buf, stc.RunStats())
    with pytest.raises(ValueError, match="exceeds cache block"):
        stc.pack_a(side, (0, 16), (0, 8), stc.BlockingParams(mc=8, nc=16, kc=8, mr=8, nr=4, kr=4), buf, stc.RunStats())
    with pytest.raises(ValueError, match="too small"):
        stc.pack_a(side, (0, 16), (0, 8), P, stc.PackedBuffer.a_panel(P, 8, 8), stc.RunStats())


def test_microkernel_properties():
    import torch

    rng = np.random.default_rng(9)
    a, b = rng.uniform(-1, 1, (8, 6)), rng.uniform(-1, 1, (6, 4))
    c0 = rng.uniform(-1, 1, 16 * 8)
    t = stc.DenseTensor((16, 8), (1, 16), torch.from_numpy(c0.copy()).cuda())
    v = stc.matrix_view(t, 8, 4)
    # k = 0 leaves the targets untouched
    stc.microkernel(a, b, 0, [(v, 0, 0, 1)], stc.RunStats())
    assert np.array_equal(bits(t.data), bits(c0))
    # +tile then -tile on integers restores C exactly; the tile equals the ordered triple loop
    ai, bi = np.round(a * 8), np.round(b * 8)
    t.data.copy_(torch.from_numpy(np.round(c0 * 8)))
    st = stc.RunStats()
    stc.microkernel(ai, bi, 6, [(v, 8, 4, 1)], st)
    acc = np.zeros((8, 4))
    for p in range(6):
        acc += np.outer(ai[:, p], bi[p])
    got = t.data.cpu().numpy().reshape(8, 16).T
    assert np.array_equal(got[8:, 4:], np.round(c0 * 8).reshape(8, 16).T[8:, 4:] + acc)
    stc.microkernel(ai, bi, 6, [(v, 8, 4, -1)], st)
    assert np.array_equal(t.data.cpu().numpy(), np.round(c0 * 8)) and st.fast_updates == 2
    # both store paths agree; PAD rows are dropped
    t.data.copy_(torch.from_numpy(c0))
    t2 = stc.DenseTensor((16, 8), (1, 16), torch.from_numpy(c0.copy()).cuda())
    s_slow = stc.RunStats()
    stc.microkernel(a, b, 6, [(v, 0, 4, 1)], stc.RunStats())
    stc.microkernel(a, b, 6, [(stc.matrix_view(t2, 8, 4), 0, 4, 1)], s_slow, force_slow=True)
    assert torch.equal(t.data, t2.data) and s_slow.slow_updates == 1
    pv = stc.pad_view(v, 24, 8)
    before = t.data.clone()
    stc.microkernel(a, b, 6, [(pv, 16, 0, 1)], stc.RunStats())
    assert torch.equal(t.data, before)
    with pytest.raises(ValueError, match="block-aligned"):
        stc.microkernel(a, b, 6, [(v, 4, 0, 1)], stc.RunStats())
    with pytest.raises(ValueError, match="do not match tile"):
        stc.microkernel(a[:4], b, 6, [(v, 0, 0, 1)], stc.RunStats())
    with pytest.raises(ValueError, match="shorter"):
        stc.microkernel(a, b, 7, [(v, 0, 0, 1)], stc.RunStats())


def test_contract_reference_is_the_classical_contraction():
    spec = stc.parse_benchmark_line("abij abef efij & a:7;b:5;i:6;j:9;e:4;f:11;")
    rm = lambda e: tuple(int(np.prod(e[i + 1:])) for i in range(len(e)))

    def tensor(labels, seed, integer):
        e = spec.tensor_extents(labels)
        rng = np.random.default_rng(seed)
        n = int(np.prod(e))
        return stc.DenseTensor(e, rm(e), rng.integers(-9, 10, n).astype(np.float64) if integer else rng.uniform(-1, 1, n))

    for integer in (True, False):
        a, b, c = tensor(spec.labels_a, 1, integer), tensor(spec.labels_b, 2, integer), tensor(spec.labels_c, 3, integer)
        ref = c.copy()
        oracle.contract_reference(spec, a, b, ref)
        assert stc.contract_reference(spec, a, b, c) is None
        if integer:
            assert np.array_equal(c.data, ref.data)
        else:
            assert oracle.relative_error(c, ref) <= 1e-14
    with pytest.raises(ValueError, match="extents"):
        stc.contract_reference(spec, a, a, c)
