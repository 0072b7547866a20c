"""Host-side planning of the host-operand pipeline (stc_host_plan, csrc/stc_host.cu): which
bundle label the problem is cut along and into how many pieces.  Pure host logic, no GPU."""

import ctypes
import os

import numpy as np
import pytest

import paper_1704_03092_b200 as stc
from paper_1704_03092_b200 import _lib
from paper_1704_03092_b200.strassen import Variant, problem_of


def _row_major(e):
    return tuple(int(np.prod(e[i + 1:])) for i in range(len(e)))


def _plan(line, level=2, c_strides=None, env=None):
    spec = stc.parse_benchmark_line(line)

    def t(labels, strides=None):
        e = spec.tensor_extents(labels)
        st = strides or _row_major(e)
        size = sum((x - 1) * s for x, s in zip(e, st)) + 1
        return stc.DenseTensor(e, st, np.zeros(size))

    p = problem_of(spec, t(spec.labels_a), t(spec.labels_b), t(spec.labels_c, c_strides), level, Variant.ABC)
    s, l, n = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    old = os.environ.get("STC_HOST_PIECES")
    if env is not None:
        os.environ["STC_HOST_PIECES"] = env
    try:
        _lib.check(_lib.lib().stc_host_plan(ctypes.byref(p), ctypes.byref(s), ctypes.byref(l), ctypes.byref(n)))
    finally:
        if env is not None:
            if old is None:
                del os.environ["STC_HOST_PIECES"]
            else:
                os.environ["STC_HOST_PIECES"] = old
    return s.value, l.value, n.value


def test_cfg2_cuts_the_i_bundle_on_a_into_four():
    # C[a,i,b,j], A[e,a,f,b]: label a has the longest runs in both A and C
    assert _plan("aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;") == (0, 0, 4)


def test_j_bundle_cut_when_its_runs_are_longer():
    # C[j,i,a,b], B[j,f,i,e]: j is outermost in both B and C
    line = "jiab eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;"
    side, label, pieces = _plan(line)
    assert (side, pieces) == (1, 4)
    assert stc.parse_benchmark_line(line).bundle_j[label] == "j"


def test_small_problems_are_not_cut():
    assert _plan("aibj eafb jfie & a:16;b:16;i:16;j:16;e:16;f:16;")[2] == 1


def test_pieces_keep_two_tiles_per_quadrant():
    # m = 1024 at L2: an I cut would leave quadrants of < 256 rows -> the J bundle (4096) is cut
    assert _plan("aibj eafb jfie & a:16;b:64;i:64;j:64;e:64;f:64;") == (1, 0, 4)
    # both bundles 1024 at L2: two pieces at most
    assert _plan("aibj eafb jfie & a:16;b:64;i:16;j:64;e:64;f:64;")[2] <= 2


def test_non_compact_c_is_not_cut():
    spec = stc.parse_benchmark_line("aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;")
    e = spec.tensor_extents(spec.labels_c)
    st = list(_row_major(e))
    st[0] += 8  # a gap after every outermost slice
    assert _plan("aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;", c_strides=tuple(st))[2] == 1


@pytest.mark.parametrize("n", ["1", "2", "8"])
def test_piece_count_override(n):
    assert _plan("aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;", env=n)[2] == int(n)


def test_host_workspace_covers_two_piece_slots():
    spec = stc.parse_benchmark_line("aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;")

    def t(labels, sp=spec):
        e = sp.tensor_extents(labels)
        return stc.DenseTensor(e, _row_major(e), np.zeros(int(np.prod(e))))

    p = problem_of(spec, t(spec.labels_a), t(spec.labels_b), t(spec.labels_c), 2, Variant.ABC)
    # one piece: the I bundle cut on a into four (a:16); it runs in the dense-M ABC
    # mode (16 tiles per term, 9 terms in flight per C tile), the whole problem ticketed
    pspec = stc.parse_benchmark_line("aibj eafb jfie & a:16;b:64;i:64;j:64;e:64;f:64;")
    pp = problem_of(pspec, t(pspec.labels_a, pspec), t(pspec.labels_b, pspec), t(pspec.labels_c, pspec), 2,
                    Variant.ABC)
    whole, host, piece = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
    L = _lib.lib()
    _lib.check(L.stc_workspace_size(ctypes.byref(p), ctypes.byref(whole)))
    _lib.check(L.stc_workspace_size(ctypes.byref(pp), ctypes.byref(piece)))
    _lib.check(L.stc_host_workspace_size(ctypes.byref(p), ctypes.byref(host)))
    assert piece.value > 49 * 256 * 1024 * 8  # the dense M slots of 49 terms
    # two piece slots + flags + the B slots the four I pieces share (49 x 1024 x 1024 doubles)
    shared_b = 49 * 1024 * 1024 * 8
    assert 2 * piece.value + shared_b <= host.value <= 2 * piece.value + shared_b + 4096 + 256


class _Stub:
    """extents / strides / base of a tensor too large to allocate (problem_of reads no data)."""

    def __init__(self, e):
        self.extents, self.strides, self.base_offset, self.data = tuple(e), _row_major(e), 0, None


def _grid(line, env=None):
    spec = stc.parse_benchmark_line(line)

    def t(labels):
        # planning reads only extents and strides: a small stand-in for the storage
        e = spec.tensor_extents(labels)
        return stc.DenseTensor(e, _row_major(e), np.zeros(int(np.prod(e)) if np.prod(e) < 1 << 22 else 1)) \
            if np.prod(e) < 1 << 22 else _Stub(e)

    p = problem_of(spec, t(spec.labels_a), t(spec.labels_b), t(spec.labels_c), 2, Variant.ABC)
    out = [ctypes.c_int32() for _ in range(4)]
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        _lib.check(_lib.lib().stc_host_grid(ctypes.byref(p), *[ctypes.byref(x) for x in out]))
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return spec, tuple(x.value for x in out)


def test_large_problems_get_an_i_by_j_grid():
    # cfg5 (24 GiB of operands): 4 x 8 pieces, the outermost label of each bundle
    spec, (la, sa, lb, sb) = _grid("abcijk abcefg efgijk & a:32;b:32;c:32;i:32;j:32;k:32;e:32;f:32;g:32;")
    assert (sa, sb) == (4, 8)
    assert spec.bundle_i[la] == "a" and spec.bundle_j[lb] == "i"
    # STC_HOST_GRID=1 keeps the 1-D cut; a forced 2 x 8 grid
    assert _grid("abcijk abcefg efgijk & a:32;b:32;c:32;i:32;j:32;k:32;e:32;f:32;g:32;",
                 {"STC_HOST_GRID": "1"})[1][1] * _grid(
        "abcijk abcefg efgijk & a:32;b:32;c:32;i:32;j:32;k:32;e:32;f:32;g:32;", {"STC_HOST_GRID": "1"})[1][3] == 8
    assert _grid("aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;", {"STC_HOST_GRID": "2x8"})[1][1::2] == (2, 8)
    # small problems stay 1-D
    _, (la, sa, lb, sb) = _grid("aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;")
    assert sa * sb == 4 and min(sa, sb) == 1


# ---- device-path planning (stc_plan_describe; host-only, grid of 148 SMs) ------------
def _describe(line, level, variant="abc"):
    import sys

    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1] / "tools"))
    from describe import describe

    return describe(line, level, variant)


@pytest.mark.parametrize("line,level,tshape,sides", [
    # cfg3 2^24, m = 256 / n = 256 at L2: 64-wide quadrants -> the narrow tiles, one-sided slots
    ("abij abef efij & a:16;b:16;i:256;j:256;e:64;f:64;", 2, 1, 1),
    ("abij abef efij & a:256;b:256;i:16;j:16;e:64;f:64;", 2, 2, 2),
    # cfg1 (576^3): 288- / 144-wide quadrants -> 128 x 64 tiles (least padding), both sides pre-summed
    ("abij abef efij & a:24;b:24;i:24;j:24;e:24;f:24;", 1, 4, 3),
    ("abij abef efij & a:24;b:24;i:24;j:24;e:24;f:24;", 2, 4, 3),
    # cfg5 and cfg2: 128 x 128 tiles, both sides pre-summed, ticketed
    ("abcijk abcefg efgijk & a:32;b:32;c:32;i:32;j:32;k:32;e:32;f:32;g:32;", 2, 0, 3),
    ("aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;", 2, 0, 3),
])
def test_plan_shapes_and_slot_sides(line, level, tshape, sides):
    info = _describe(line, level)
    assert info["tshape"] == tshape, info
    assert info["presum"] == 1 and info["presum_sides"] == sides, info
    if tshape in (1, 2, 3, 4):
        assert info["ticketed"] == 0, info  # the narrow / small shapes write dense M
    assert info["terms"] == 7 ** level


def test_sharded_workspace_covers_every_shard():
    # stc_sharded_workspace_size: at least each shard's own stc_workspace_size (host-only)
    spec = stc.parse_benchmark_line("abij abef efij & a:8;b:16;i:12;j:16;e:8;f:16;")

    def t(labels):
        e = spec.tensor_extents(labels)
        return stc.DenseTensor(e, _row_major(e), np.zeros(int(np.prod(e))))

    p = problem_of(spec, t(spec.labels_a), t(spec.labels_b), t(spec.labels_c), 2, Variant.ABC)
    L = _lib.lib()
    need = ctypes.c_size_t()
    _lib.check(L.stc_sharded_workspace_size(ctypes.byref(p), 3, -1, ctypes.byref(need)))
    for rank in range(3):
        q = _lib.Problem()
        _lib.check(L.stc_shard_problem(ctypes.byref(p), 3, rank, -1, ctypes.byref(q), None, None, None))
        each = ctypes.c_size_t()
        _lib.check(L.stc_workspace_size(ctypes.byref(q), ctypes.byref(each)))
        assert need.value >= each.value
    with pytest.raises(ValueError):
        _lib.check(L.stc_sharded_workspace_size(ctypes.byref(p), 0, -1, ctypes.byref(need)))


@pytest.mark.parametrize("line,grid", [
    # cfg5 (24 GiB, J 32768 wide): 4 x 8; its shards of 4 and 2 GPUs (14 / 20 GiB, J 8192 /
    # 16384 wide): 4 x 4 (a J cut in 8 only while the pieces stay >= 4096 wide)
    ("abcijk abcefg efgijk & a:32;b:32;c:32;i:32;j:32;k:32;e:32;f:32;g:32;", (4, 8)),
    ("abcijk abcefg efgijk & a:32;b:32;c:32;i:8;j:32;k:32;e:32;f:32;g:32;", (4, 4)),
    ("abcijk abcefg efgijk & a:32;b:32;c:32;i:16;j:32;k:32;e:32;f:32;g:32;", (4, 4)),
])
def test_host_grid_shapes(line, grid):
    _, (la, sa, lb, sb) = _grid(line)
    assert (sa, sb) == grid


def test_host_one_d_cut_in_eight_from_4_gb():
    # the cfg5 shard of 8 GPUs (11 GiB: below the grid threshold): 8 pieces along I
    spec = stc.parse_benchmark_line("abcijk abcefg efgijk & a:32;b:32;c:32;i:4;j:32;k:32;e:32;f:32;g:32;")
    t = lambda labels: _Stub(spec.tensor_extents(labels))  # noqa: E731
    p = problem_of(spec, t(spec.labels_a), t(spec.labels_b), t(spec.labels_c), 2, Variant.ABC)
    side, label, pieces = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _lib.check(_lib.lib().stc_host_plan(ctypes.byref(p), ctypes.byref(side), ctypes.byref(label), ctypes.byref(pieces)))
    assert (side.value, pieces.value) == (0, 8)
