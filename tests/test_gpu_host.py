"""GPU parity of the host-operand entry point (stc_contract_host, stc_host.cu).

Host operands are uploaded, contracted piece by piece (the I or J bundle cut
along one label) and downloaded with the transfers pipelined against the DMMA
work.  Checks, against the CPU oracle's classical contraction:
  * integer-valued data: exact for every piece count, variant and level;
  * random data: normwise error <= 1e-12 (the reference suite's bound);
  * J-side splits, pinned and pageable storage, base offsets and a
    non-compact C (which disables the split);
  * the staged path (STC_HOST_PIPELINE=0) agrees.
"""

import ctypes
import os

import numpy as np
import pytest

import oracle
import paper_1704_03092_b200 as stc
from paper_1704_03092_b200 import _lib
from paper_1704_03092_b200.strassen import Variant, problem_of

pytestmark = pytest.mark.gpu

TOL = 1e-12
# I bundle split on a (A and C), J bundle split on j (B outermost j; C: j ahead of i)
LINES = {
    "i_split": "aibj eafb jfie & a:32;b:64;i:16;j:64;e:32;f:32;",
    "j_split": "jiab eafb jfie & a:16;b:64;i:32;j:64;e:32;f:32;",
}


def _row_major(e):
    return tuple(int(np.prod(e[i + 1:])) for i in range(len(e)))


def _tensor(spec, labels, seed, ints, pad=0):
    e = spec.tensor_extents(labels)
    n = int(np.prod(e))
    rng = np.random.default_rng(seed)
    data = rng.integers(-8, 9, n + pad).astype(np.float64) if ints else rng.uniform(-1, 1, n + pad)
    return stc.DenseTensor(e, _row_major(e), data, pad)


def _plan(spec, a, b, c, level):
    p = problem_of(spec, a, b, c, level, Variant.ABC)
    s, l, n = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _lib.check(_lib.lib().stc_host_plan(ctypes.byref(p), ctypes.byref(s), ctypes.byref(l), ctypes.byref(n)))
    return s.value, l.value, n.value


def _with_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.mark.parametrize("name", sorted(LINES))
def test_host_pipeline_integer_exact(name):
    spec = stc.parse_benchmark_line(LINES[name])
    a, b, c0 = (_tensor(spec, l, s, True) for l, s in ((spec.labels_a, 1), (spec.labels_b, 2), (spec.labels_c, 3)))
    ref = c0.copy()
    oracle.contract_reference(spec, a, b, ref, threads=8)
    side = {"i_split": 0, "j_split": 1}[name]
    for pieces in ("1", "2", "4"):
        assert _with_env({"STC_HOST_PIECES": pieces}, lambda: _plan(spec, a, b, c0, 2))[::2] == \
            ((side if pieces != "1" else 0), int(pieces))
        for level in (0, 1, 2):
            for variant in ("abc", "ab", "naive"):
                c = c0.copy()
                st = _with_env({"STC_HOST_PIECES": pieces}, lambda: stc.contract(spec, a, b, c, level, variant))
                assert st.leaf_multiplies == 7 ** level
                assert np.array_equal(c.data, ref.data), (pieces, level, variant)


def test_host_pipeline_random_pinned_and_offsets():
    import torch

    spec = stc.parse_benchmark_line(LINES["i_split"])
    a, b, c0 = (_tensor(spec, l, s, False, pad=3) for l, s in ((spec.labels_a, 4), (spec.labels_b, 5),
                                                              (spec.labels_c, 6)))
    ref = c0.copy()
    oracle.contract_reference(spec, a, b, ref, threads=8)
    outs = []
    for pinned in (False, True):
        for env in ({}, {"STC_HOST_PIECES": "8"}, {"STC_HOST_PIPELINE": "0"}):
            c = c0.copy()
            aa, bb = a, b
            if pinned:
                aa, bb, c = (stc.DenseTensor(t.extents, t.strides, torch.from_numpy(t.data).pin_memory(),
                                             t.base_offset) for t in (a, b, c))
            _with_env(env, lambda: stc.contract(spec, aa, bb, c, 2, "abc"))
            got = c.data.numpy() if torch.is_tensor(c.data) else c.data
            assert np.array_equal(got[:3], c0.data[:3])  # storage ahead of base_offset untouched
            outs.append(got)
            err = np.linalg.norm(got - ref.data) / np.linalg.norm(ref.data)
            assert err <= TOL, (pinned, env, err)
    for o in outs[1:]:
        assert np.array_equal(o, outs[0]) or np.linalg.norm(o - outs[0]) / np.linalg.norm(outs[0]) <= TOL


def test_host_pipeline_non_compact_c_is_not_split():
    # C stored with a gap between its rows: not compact, so one piece; the gap is preserved
    spec = stc.parse_benchmark_line(LINES["i_split"])
    a, b = _tensor(spec, spec.labels_a, 7, True), _tensor(spec, spec.labels_b, 8, True)
    e = spec.tensor_extents(spec.labels_c)
    strides = list(_row_major(e))
    strides[0] += 5  # gap after every outermost slice
    size = (e[0] - 1) * strides[0] + strides[1] * e[1]
    data = np.random.default_rng(9).integers(-8, 9, size).astype(np.float64)
    c0 = stc.DenseTensor(e, tuple(strides), data)
    assert _plan(spec, a, b, c0, 2)[2] == 1
    ref = c0.copy()
    oracle.contract_reference(spec, a, b, ref, threads=8)
    c = c0.copy()
    stc.contract(spec, a, b, c, 2, "abc")
    assert np.array_equal(c.data, ref.data)


def test_host_pipeline_irregular_pieces_integer_exact():
    # odd extents: pieces of 25 along a (PAD quadrants, repacked operands)
    spec = stc.parse_benchmark_line("abcij eafbc ifje & a:50;b:7;c:13;i:14;j:9;e:18;f:11;")
    a, b, c0 = (_tensor(spec, l, s, True) for l, s in ((spec.labels_a, 11), (spec.labels_b, 12), (spec.labels_c, 13)))
    ref = c0.copy()
    oracle.contract_reference(spec, a, b, ref, threads=8)
    for pieces in ("2", "5"):
        for level, variant in ((1, "abc"), (2, "abc"), (2, "ab"), (2, "naive")):
            c = c0.copy()
            _with_env({"STC_HOST_PIECES": pieces}, lambda: stc.contract(spec, a, b, c, level, variant))
            assert np.array_equal(c.data, ref.data), (pieces, level, variant)


def test_host_pipeline_torch_cpu_storage_and_validate():
    import torch

    spec = stc.parse_benchmark_line(LINES["j_split"])
    a, b, c0 = (_tensor(spec, l, s, True) for l, s in ((spec.labels_a, 14), (spec.labels_b, 15), (spec.labels_c, 16)))
    ref = c0.copy()
    oracle.contract_reference(spec, a, b, ref, threads=8)
    ta, tb, tc = (stc.DenseTensor(t.extents, t.strides, torch.from_numpy(t.data.copy()), t.base_offset)
                  for t in (a, b, c0))
    st = stc.contract(spec, ta, tb, tc, 2, "abc", validate=True)
    assert st.leaf_multiplies == 49 and st.seconds > 0
    assert np.array_equal(tc.data.numpy(), ref.data)


def test_host_pipeline_errors_leave_c_untouched():
    # C-ABI errors come before any transfer: C's host storage is unchanged
    import torch

    spec = stc.parse_benchmark_line(LINES["i_split"])
    a, b, c0 = (_tensor(spec, l, s, False) for l, s in ((spec.labels_a, 17), (spec.labels_b, 18), (spec.labels_c, 19)))
    c = c0.copy()
    p = problem_of(spec, a, b, c, 2, Variant.ABC)
    p.c_row.ext[0] += 1  # I extents of A and C differ
    L = _lib.lib()
    d = [torch.empty(t.data.size + 64, dtype=torch.float64, device="cuda") for t in (a, b, c)]
    ws = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    rc = L.stc_contract_host(ctypes.byref(p), ctypes.c_void_p(a.data.ctypes.data), ctypes.c_void_p(b.data.ctypes.data),
                             ctypes.c_void_p(c.data.ctypes.data), *(ctypes.c_void_p(x.data_ptr()) for x in d),
                             ctypes.c_void_p(ws.data_ptr()), ws.numel(), None, None)
    torch.cuda.synchronize()
    assert rc == _lib.STC_EINVAL and b"extents" in L.stc_last_error()
    assert np.array_equal(c.data, c0.data)
    # workspace too small
    p = problem_of(spec, a, b, c, 2, Variant.ABC)
    rc = L.stc_contract_host(ctypes.byref(p), ctypes.c_void_p(a.data.ctypes.data), ctypes.c_void_p(b.data.ctypes.data),
                             ctypes.c_void_p(c.data.ctypes.data), *(ctypes.c_void_p(x.data_ptr()) for x in d),
                             ctypes.c_void_p(ws.data_ptr()), 256, None, None)
    assert rc == _lib.STC_EWORKSPACE
    assert np.array_equal(c.data, c0.data)


def _pinned(t):
    import torch

    return stc.DenseTensor(t.extents, t.strides, torch.from_numpy(t.data).pin_memory(), t.base_offset)


@pytest.mark.parametrize("pieces", ["2", "4"])
def test_host_pipeline_pieces_against_device_path(pieces):
    # host operands: the problem is cut into pieces, each its own L-level Strassen over
    # its own quadrants (a different pairing than the whole problem: rounding-level
    # differences only); RunStats reports the piece count beside leaf_multiplies = 7^L
    import torch

    spec = stc.parse_benchmark_line("aibj eafb jfie & a:32;b:64;i:32;j:64;e:32;f:32;")
    a, b, c0 = (_tensor(spec, l, s, False) for l, s in ((spec.labels_a, 7), (spec.labels_b, 8), (spec.labels_c, 9)))
    dev = stc.DenseTensor(c0.extents, c0.strides, torch.from_numpy(c0.data.copy()).cuda(), 0)
    sd = stc.contract(spec, a.to_device(), b.to_device(), dev, 2, "abc")
    assert sd.pieces == 1
    want = dev.data.cpu().numpy()
    ha, hb, hc = _pinned(a), _pinned(b), _pinned(c0.copy())
    st = _with_env({"STC_HOST_PIECES": pieces}, lambda: stc.contract(spec, ha, hb, hc, 2, "abc"))
    assert st.pieces == int(pieces) and st.leaf_multiplies == 49, st
    assert np.linalg.norm(hc.data.numpy() - want) / np.linalg.norm(want) <= TOL
    ref = c0.copy()
    oracle.contract_reference(spec, a, b, ref, threads=oracle.max_threads())
    got = stc.DenseTensor(c0.extents, c0.strides, hc.data.numpy())
    assert oracle.relative_error(got, ref) <= TOL


@pytest.mark.parametrize("level,variant", [(1, "abc"), (2, "naive")])
def test_host_operands_with_negative_strides(level, variant):
    # the reference's DenseTensor allows negative strides (tensor.py:43-97): a reversed
    # numpy view as A and as C, host storage, through the host pipeline
    spec = stc.parse_benchmark_line("abij abef efij & a:7;b:6;i:5;j:9;e:4;f:8;")
    a, b, c0 = (_tensor(spec, l, s, False) for l, s in ((spec.labels_a, 3), (spec.labels_b, 4), (spec.labels_c, 5)))

    def reversed_first_axis(t):
        st = list(t.strides)
        base = t.base_offset + (t.extents[0] - 1) * st[0]
        st[0] = -st[0]
        # the same elements addressed from the other end: value at index i is the old (n-1-i)
        return stc.DenseTensor(t.extents, tuple(st), t.data.copy(), base)

    ra, rc = reversed_first_axis(a), reversed_first_axis(c0)
    ref = rc.copy()
    oracle.contract_reference(spec, ra, b, ref)
    got = rc.copy()
    st = stc.contract(spec, ra, b, got, level, variant)
    assert st.leaf_multiplies == 7 ** level
    assert oracle.relative_error(got, ref) <= TOL


@pytest.mark.parametrize("grid", ["2x2", "2x4", "4x2"])
def test_host_grid_pieces_integer_exact(grid):
    # the I x J grid of host pieces (large problems' default, forced here): each piece an
    # independent contraction of its (I range, J range) block; integer data -> exact
    spec = stc.parse_benchmark_line("abcijk abcefg efgijk & a:8;b:6;c:4;i:8;j:6;k:4;e:4;f:6;g:8;")
    a, b, c0 = (_tensor(spec, l, s, True) for l, s in ((spec.labels_a, 21), (spec.labels_b, 22), (spec.labels_c, 23)))
    ref = c0.copy()
    oracle.contract_reference(spec, a, b, ref, threads=8)
    for level, variant in ((1, "abc"), (2, "abc"), (2, "ab"), (2, "naive")):
        c = _pinned(c0.copy())
        st = _with_env({"STC_HOST_GRID": grid}, lambda: stc.contract(spec, _pinned(a), _pinned(b), c, level, variant))
        sa, sb = (int(x) for x in grid.split("x"))
        # (up to +3: the first cell may run as 2 or 4 k parts, STC_HOST_KSPLIT)
        assert sa * sb <= st.pieces <= sa * sb + 3 and st.leaf_multiplies == 7 ** level, st
        assert np.array_equal(c.data.numpy(), ref.data), (grid, level, variant)


@pytest.mark.parametrize("grid", ["2x2", "4x2", "4x4", "pieces4"])
def test_host_grid_shared_slots_match_unshared_bitwise(grid):
    # pieces of a grid that pre-sum both sides share the slots of their A rows / B columns
    # (formed once by the first piece of each); the C blocks must equal those of pieces
    # that form their own slots, bit for bit, and the oracle's classical result
    spec = stc.parse_benchmark_line("abij abef efij & a:32;b:16;i:32;j:16;e:32;f:16;")
    a, b, c0 = (_tensor(spec, l, s, False) for l, s in ((spec.labels_a, 31), (spec.labels_b, 32), (spec.labels_c, 33)))
    ref = c0.copy()
    oracle.contract_reference(spec, a, b, ref, threads=oracle.max_threads())
    for level, variant in ((2, "abc"), (1, "abc"), (2, "ab")):
        outs = []
        for share in ("1", "0"):
            c = _pinned(c0.copy())
            # (pieces4: a 1-D cut into 4 pieces, sharing the operand the pieces use whole)
            split = {"STC_HOST_PIECES": "4"} if grid == "pieces4" else {"STC_HOST_GRID": grid}
            env = {**split, "STC_PRESUM_OPS": "1", "STC_HOST_SHARE": share}
            st = _with_env(env, lambda: stc.contract(spec, _pinned(a), _pinned(b), c, level, variant))
            sa, sb = (4, 1) if grid == "pieces4" else (int(x) for x in grid.split("x"))
            assert sa * sb <= st.pieces <= sa * sb + 3 and st.leaf_multiplies == 7 ** level, st
            outs.append(c.data.numpy().copy())
        assert np.array_equal(outs[0], outs[1]), (grid, level, variant)
        got = stc.DenseTensor(c0.extents, c0.strides, outs[0])
        assert oracle.relative_error(got, ref) <= TOL
