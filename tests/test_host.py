"""Host-side logic of the drop-in package (no GPU needed): the data model, the
benchmark-line grammar, the Strassen term table, argument validation and the
C-ABI library surface.  Mirrors pkg/tests/test_tensor.py and the table tests
of pkg/tests/test_strassen.py."""

import pathlib
import re

import numpy as np
import pytest

import golden_io
import paper_1704_03092_b200 as stc
from paper_1704_03092_b200 import _lib

ROOT = pathlib.Path(__file__).resolve().parents[1]


def test_parse_appendix_line():
    spec = stc.parse_benchmark_line("abc dca db & a:4;b:8;c:2;d:8;")
    assert (spec.labels_c, spec.labels_a, spec.labels_b) == ("abc", "dca", "db")
    assert (spec.bundle_i, spec.bundle_j, spec.bundle_p) == ("ac", "b", "d")
    assert (spec.n_i, spec.n_j, spec.n_p) == (8, 8, 8)
    assert stc.to_benchmark_line(spec) == "abc dca db & a:4;b:8;c:2;d:8;"


def test_parse_trailing_semicolon_optional():
    assert stc.parse_benchmark_line("ab ac cb & a:2;b:3;c:4") == stc.parse_benchmark_line("ab ac cb & a:2;b:3;c:4;")


@pytest.mark.parametrize(
    "line, message",
    [
        ("abc dca db a:4;b:8;c:2;d:8;", "separator"),
        ("abc dca & a:4;b:8;c:2;d:8;", "three label groups"),
        ("abc dca db & a:4;b:8;c:2;", "missing extent"),
        ("abc dca db & a:4;b:8;c:2;d:8;z:1;", "unknown label"),
        ("abc dca dbe & a:4;b:8;c:2;d:8;e:2;", "one tensor only"),
        ("ab ab ab & a:2;b:2;", "all three"),
        ("ab ac cb & a:0;b:2;c:2;", "non-positive"),
        ("aab ac cb & a:2;b:2;c:2;", "repeated label"),
        ("a1 ac cb & a:2;c:2;", "single ASCII"),
        ("ab ac cb & a:two;b:2;c:2;", "malformed extent"),
        ("ab ac cb & a:2;a:2;b:2;c:2;", "duplicate extent"),
    ],
)
def test_parse_errors_keep_reference_keywords(line, message):
    with pytest.raises(stc.BenchmarkParseError, match=message):
        stc.parse_benchmark_line(line)


def test_round_trip_on_golden_specs():
    meta, _ = golden_io.contract_cases()
    for m in meta:
        spec = stc.parse_benchmark_line(m["line"])
        assert stc.parse_benchmark_line(stc.to_benchmark_line(spec)) == spec
        assert stc.to_benchmark_line(spec) == m["line"]


def test_read_benchmark_file(tmp_path):
    f = tmp_path / "b.txt"
    f.write_text("# comment\n\nab ac cb & a:2;b:3;c:4;\nabc dca db & a:4;b:8;c:2;d:8;\n")
    assert len(stc.read_benchmark_file(f)) == 2
    f.write_text("ab ac cb & a:2;b:3;c:4;\nab ac & a:1;\n")
    with pytest.raises(stc.BenchmarkParseError, match=":2:"):
        stc.read_benchmark_file(f)


def test_dense_tensor_model():
    t = stc.make_dense_tensor((2, 3, 4), "sequence")
    assert t.strides == (1, 2, 6) and t.size == 24
    assert stc.element_at(t, (1, 2, 3)) == 1 + 2 * 2 + 3 * 6
    stc.set_element(t, (0, 0, 0), 7.0)
    assert t.data[0] == 7.0
    with pytest.raises(ValueError, match="out of bounds"):
        stc.DenseTensor((3, 3), (1, 3), np.zeros(8))
    with pytest.raises(ValueError, match="positive"):
        stc.make_dense_tensor((0, 2))
    r1, r2 = stc.make_dense_tensor((5, 5), "random", 3), stc.make_dense_tensor((5, 5), "random", 3)
    assert np.array_equal(r1.data, r2.data)
    assert np.array_equal(r1.data, np.random.default_rng(3).uniform(-1, 1, 25))


def test_strassen_terms_match_reference_golden():
    terms = golden_io.terms()
    for level in range(4):
        got = [[list(map(list, t.a_ops)), list(map(list, t.b_ops)), list(map(list, t.c_ops))]
               for t in stc.strassen_terms(level, allow_deep=True)]
        assert got == terms[str(level)]


def test_level_cap_and_validation():
    with pytest.raises(ValueError):
        stc.strassen_terms(-1)
    with pytest.raises(ValueError, match="cap"):
        stc.strassen_terms(3)
    assert len(stc.strassen_terms(3, allow_deep=True)) == 343


def test_quadrant_rc_row_major_top_level_most_significant():
    # level 1: 0=TL 1=TR 2=BL 3=BR
    assert [stc.quadrant_rc(q, 1) for q in range(4)] == [(0, 0), (0, 1), (1, 0), (1, 1)]
    # level 2: id = q1*4 + q2, row = 2*r1 + r2
    assert stc.quadrant_rc(13, 2) == (2, 3) and stc.quadrant_rc(6, 2) == (1, 2)


def test_contract_errors_before_any_device_work():
    spec = stc.parse_benchmark_line("ab ac cb & a:4;b:4;c:4;")
    bad = stc.make_dense_tensor((4, 5))
    with pytest.raises(ValueError, match="extents"):
        stc.contract(spec, bad, stc.make_dense_tensor((4, 4)), stc.make_dense_tensor((4, 4)), 1, "abc")
    ok = stc.make_dense_tensor((4, 4))
    with pytest.raises(ValueError, match="cap"):
        stc.contract(spec, ok, ok.copy(), ok.copy(), 3, "abc")


def test_blocking_params_validation():
    with pytest.raises(ValueError, match="multiples"):
        stc.BlockingParams(mc=10, mr=8)
    with pytest.raises(ValueError, match="positive"):
        stc.BlockingParams(kr=0)


def test_effective_gflops_identity():
    assert stc.effective_gflops(1000, 1000, 1000, 0.1) == pytest.approx(20.0, rel=1e-15)
    with pytest.raises(ValueError):
        stc.effective_gflops(8, 8, 8, 0.0)


def test_problem_descriptor_bundles():
    spec = stc.parse_benchmark_line("aibj eafb jfie & a:3;b:4;i:5;j:6;e:7;f:2;")
    ext_a, ext_b, ext_c = (spec.tensor_extents(spec.labels_a), spec.tensor_extents(spec.labels_b),
                           spec.tensor_extents(spec.labels_c))
    rm = lambda e: tuple(int(np.prod(e[i + 1:])) for i in range(len(e)))
    a = stc.DenseTensor(ext_a, rm(ext_a), np.zeros(int(np.prod(ext_a))), 0)
    b = stc.DenseTensor(ext_b, rm(ext_b), np.zeros(int(np.prod(ext_b))), 0)
    c = stc.DenseTensor(ext_c, rm(ext_c), np.zeros(int(np.prod(ext_c))), 0)
    p = stc.strassen.problem_of(spec, a, b, c, 2, stc.Variant.ABC)
    # I = (a, b) in C order; A = [e, a, f, b]
    assert p.a_row.nlab == 2 and list(p.a_row.ext[:2]) == [3, 4] and list(p.a_row.str[:2]) == [a.strides[1], a.strides[3]]
    # P = (e, f) in A order; B = [j, f, i, e]
    assert list(p.b_row.ext[:2]) == [7, 2] and list(p.b_row.str[:2]) == [b.strides[3], b.strides[1]]
    # J = (i, j) in C order
    assert list(p.c_col.ext[:2]) == [5, 6] and list(p.c_col.str[:2]) == [c.strides[1], c.strides[3]]
    assert p.level == 2 and p.variant == 0


def _header_symbols():
    text = (ROOT / "include" / "stc_b200.h").read_text()
    return sorted(set(re.findall(r"\b(stc_[a-z_]+)\s*\(", text)))


def test_c_abi_library_exports_every_header_symbol():
    import ctypes

    lib = _lib.lib()  # loads libstc_b200.so (no GPU needed to load)
    syms = _header_symbols()
    assert len(syms) >= 12
    for name in syms:
        assert hasattr(lib, name), name
        assert name in _lib.exported_symbols(), name
    assert lib.stc_abi_version() == 1
    # host-only entry point: workspace sizing works without a GPU
    spec = stc.parse_benchmark_line("ab ac cb & a:300;b:200;c:100;")
    t = lambda e: stc.DenseTensor(e, (1, e[0]), np.zeros(int(np.prod(e))))
    p = stc.strassen.problem_of(spec, t((300, 100)), t((100, 200)), t((300, 200)), 2, stc.Variant.ABC)
    need = ctypes.c_size_t()
    assert lib.stc_workspace_size(ctypes.byref(p), ctypes.byref(need)) == 0 and need.value > 0
    p.level = 7
    with pytest.raises(ValueError, match="cap"):
        _lib.check(lib.stc_workspace_size(ctypes.byref(p), ctypes.byref(need)))


def test_component_entries_reject_bad_arguments_before_device_work():
    """stc_pack_panel / stc_microtile validate on the host (no GPU needed to fail)."""
    import ctypes

    lib = _lib.lib()
    P = ctypes.POINTER
    one = (ctypes.c_void_p * 1)(8)
    pp = ctypes.cast(one, P(ctypes.c_void_p))
    co = (ctypes.c_double * 1)(1.0)
    dummy = ctypes.c_void_p(256)

    def pack(side=0, nviews=1, x0=0, k0=0, width=8, kblock=4, depth=8, coeff=1.0):
        co[0] = coeff
        return lib.stc_pack_panel(side, dummy, nviews, pp, pp, None, None, co, x0, 16, k0, 8, width, kblock, 0, dummy,
                                  depth, None, None)

    for kw, word in ((dict(side=2), "side"), (dict(nviews=0), "views"), (dict(nviews=17), "views"),
                     (dict(x0=4), "multiple"), (dict(k0=2), "multiple"), (dict(depth=4), "invalid"),
                     (dict(width=0), "invalid"), (dict(coeff=2.0), r"\+/-1")):
        with pytest.raises(ValueError, match=word):
            _lib.check(pack(**kw))
    i64 = lambda v: (ctypes.c_int64 * 1)(v)

    def micro(k=4, mr=8, nr=4, lda=4, ldb=4, ntg=1, i0=0, j0=0, m=16, n=8):
        return lib.stc_microtile(dummy, lda, dummy, ldb, k, mr, nr, dummy, ntg, pp, pp, None, None, co, i64(i0), i64(j0),
                                 i64(m), i64(n), 0, None, None)

    assert micro(k=0) == 0  # k = 0: nothing to do (kernels.py:211-212)
    for kw, word in ((dict(lda=3), "invalid"), (dict(ldb=3), "invalid"), (dict(mr=0), "invalid"),
                     (dict(ntg=17), "targets"), (dict(i0=4), "block-aligned"), (dict(j0=2), "block-aligned"),
                     (dict(i0=16), "outside")):
        with pytest.raises(ValueError, match=word):
            _lib.check(micro(**kw))


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle (test infrastructure)."""
    for f in (ROOT / "paper_1704_03092_b200").glob("*.py"):
        assert "import oracle" not in f.read_text() and "from oracle" not in f.read_text(), f
