"""GPU parity: the sm_100a path against the reference's own outputs (golden
fixtures) and the CPU oracle, through the public API (which calls the C ABI).

Tolerances: floating-point cases <= 1e-12 normwise relative error against the
reference output of the same level and variant and against the classical
result (the reference suite's own bound, pkg/tests/test_acceptance.py:157-165;
the north star's gate is 1e-10).  Integer cases: bitwise.
"""

import numpy as np
import pytest

import golden_io
import oracle
import paper_1704_03092_b200 as stc

pytestmark = pytest.mark.gpu

TOL = 1e-12
META, ARR = golden_io.contract_cases()
CASES = list(range(len(META)))


@pytest.mark.parametrize("k", CASES)
def test_golden_contract_all_levels_variants(k):
    spec = stc.parse_benchmark_line(META[k]["line"])
    a, b, c0 = golden_io.case_operands(stc.DenseTensor, META, ARR, k)
    classical = stc.DenseTensor(c0.extents, c0.strides, ARR[f"k{k}_classical"])
    for run in META[k]["runs"]:
        level, variant = run["level"], run["variant"]
        c = c0.copy()
        st = stc.contract(spec, a, b, c, level, variant)
        ref = stc.DenseTensor(c0.extents, c0.strides, ARR[f"k{k}_L{level}_{variant}"])
        assert st.leaf_multiplies == 7 ** level
        if META[k]["fill"] == "int":
            assert np.array_equal(c.data, ref.data), (level, variant)
            assert np.array_equal(c.data, classical.data), (level, variant)
        else:
            assert stc.relative_error(c, ref) <= TOL, (level, variant)
            assert stc.relative_error(c, classical) <= TOL, (level, variant)


@pytest.mark.parametrize("k", CASES[:6])
def test_device_resident_operands_match_host_staged(k):
    import torch

    spec = stc.parse_benchmark_line(META[k]["line"])
    a, b, c0 = golden_io.case_operands(stc.DenseTensor, META, ARR, k)
    c_host = c0.copy()
    stc.contract(spec, a, b, c_host, 2, "abc")
    cd = c0.to_device()
    stc.contract(spec, a.to_device(), b.to_device(), cd, 2, "abc")
    torch.cuda.synchronize()
    assert np.array_equal(cd.data.cpu().numpy(), c_host.data)


def test_force_slow_and_reference_tiling_are_bitwise_neutral():
    spec = stc.parse_benchmark_line("abcd aebf dfce & a:8;b:16;c:16;d:8;e:16;f:16;")
    a = stc.make_dense_tensor(spec.tensor_extents(spec.labels_a), "random", 1)
    b = stc.make_dense_tensor(spec.tensor_extents(spec.labels_b), "random", 2)
    c0 = stc.make_dense_tensor(spec.tensor_extents(spec.labels_c), "random", 3)
    for level in (0, 1, 2):
        outs = []
        for kw in ({}, {"force_slow": True}):
            c = c0.copy()
            stc.contract(spec, a, b, c, level, "abc", **kw)
            outs.append(c.data)
        assert np.array_equal(outs[0], outs[1])


def test_run_to_run_bitwise_determinism():
    spec = stc.parse_benchmark_line("abij abef efij & a:16;b:24;i:20;j:16;e:24;f:12;")
    a = stc.make_dense_tensor(spec.tensor_extents(spec.labels_a), "random", 4)
    b = stc.make_dense_tensor(spec.tensor_extents(spec.labels_b), "random", 5)
    c0 = stc.make_dense_tensor(spec.tensor_extents(spec.labels_c), "random", 6)
    for variant in stc.Variant:
        outs = []
        for _ in range(3):
            c = c0.copy()
            stc.contract(spec, a, b, c, 2, variant)
            outs.append(c.data)
        assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_accumulation_semantics_twice():
    spec = stc.parse_benchmark_line("ab ac cb & a:40;b:36;c:44;")
    a = stc.make_dense_tensor((40, 44), "random", 31)
    b = stc.make_dense_tensor((44, 36), "random", 32)
    c0 = stc.make_dense_tensor((40, 36), "random", 33)
    c = c0.copy()
    stc.contract(spec, a, b, c, 1, "abc")
    stc.contract(spec, a, b, c, 1, "abc")
    ref = c0.copy()
    oracle.contract_reference(spec, a, b, ref)
    oracle.contract_reference(spec, a, b, ref)
    assert oracle.relative_error(c, ref) <= TOL


def test_level_three_allow_deep():
    spec = stc.parse_benchmark_line("ab ac cb & a:20;b:18;c:22;")
    a = stc.make_dense_tensor((20, 22), "random", 41)
    b = stc.make_dense_tensor((22, 18), "random", 42)
    c0 = stc.make_dense_tensor((20, 18), "random", 43)
    with pytest.raises(ValueError, match="cap"):
        stc.contract(spec, a, b, c0.copy(), 3, "abc")
    ref = c0.copy()
    oracle.contract_reference(spec, a, b, ref)
    for variant in stc.Variant:
        c = c0.copy()
        st = stc.contract(spec, a, b, c, 3, variant, allow_deep=True)
        assert st.leaf_multiplies == 343
        assert oracle.relative_error(c, ref) <= TOL


def test_cfg1_against_reference_l1_abc():
    """BASELINE config 1 at full size against the reference's own L1 ABC output."""
    g = golden_io.cfg1()
    spec = stc.parse_benchmark_line(g["line"])
    ext = (24, 24, 24, 24)
    rm = (24 ** 3, 24 ** 2, 24, 1)
    a = stc.DenseTensor(ext, rm, np.random.default_rng(g["seed_a"]).uniform(-1, 1, 24 ** 4))
    b = stc.DenseTensor(ext, rm, np.random.default_rng(g["seed_b"]).uniform(-1, 1, 24 ** 4))
    c = stc.DenseTensor(ext, rm, np.zeros(24 ** 4))
    st = stc.contract(spec, a, b, c, 1, "abc")
    assert st.leaf_multiplies == 7
    idx = np.asarray(g["sample_index"])
    ref = np.asarray(g["sample_value"])
    assert np.linalg.norm(c.data[idx] - ref) / np.linalg.norm(ref) <= TOL
    assert abs(np.sqrt(np.sum(c.data ** 2)) - g["frob"]) / g["frob"] <= TOL
    # and the whole tensor against the bitwise-pinned oracle port of the same variant
    c2 = stc.DenseTensor(ext, rm, np.zeros(24 ** 4))
    oracle.contract(spec, a, b, c2, 1, "abc", threads=oracle.max_threads())
    assert oracle.relative_error(c, c2) <= TOL
