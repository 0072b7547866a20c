"""The CPU oracle (oracle/stc_oracle.c) pinned against the REFERENCE's own outputs.

The fixtures in tests/golden/ were produced by running the reference package
(tests/golden/make_golden.py).  The oracle restates the reference algorithm in C
with the same accumulation order, so every comparison here is bitwise.
"""

import json

import numpy as np
import pytest

import golden_io
import oracle

META, ARR = golden_io.contract_cases()


class _T:
    """Minimal DenseTensor stand-in (the oracle is duck-typed)."""

    def __init__(self, extents, strides, data, base_offset=0):
        self.extents, self.strides, self.data, self.base_offset = tuple(extents), tuple(strides), data, base_offset

    def copy(self):
        return _T(self.extents, self.strides, self.data.copy(), self.base_offset)


class _Spec:
    def __init__(self, line):
        head, tail = line.split("&")
        self.labels_c, self.labels_a, self.labels_b = head.split()
        self.extents = {kv.split(":")[0].strip(): int(kv.split(":")[1]) for kv in tail.split(";") if kv.strip()}

    def tensor_extents(self, labels):
        return tuple(self.extents[l] for l in labels)


def _operands(k):
    return golden_io.case_operands(_T, META, ARR, k)


@pytest.mark.parametrize("k", range(len(META)))
def test_oracle_contract_is_bitwise_the_reference(k):
    spec = _Spec(META[k]["line"])
    a, b, c0 = _operands(k)
    for run in META[k]["runs"]:
        c = c0.copy()
        st = oracle.contract(spec, a, b, c, run["level"], run["variant"])
        assert np.array_equal(c.data, ARR[f"k{k}_L{run['level']}_{run['variant']}"]), run
        assert st["leaf_multiplies"] == run["leaf"] == 7 ** run["level"]
        assert st["total_flops"] == run["total_flops"]
        for key in ("fast_blocks", "slow_blocks", "fast_updates", "slow_updates"):
            assert st[key] == run[key], (key, run)


@pytest.mark.parametrize("k", range(len(META)))
def test_oracle_classical_is_bitwise_the_reference(k):
    spec = _Spec(META[k]["line"])
    a, b, c0 = _operands(k)
    c = c0.copy()
    oracle.contract_reference(spec, a, b, c)
    assert np.array_equal(c.data, ARR[f"k{k}_classical"])


def test_oracle_relative_error_matches_reference_values():
    for k in range(len(META)):
        spec = _Spec(META[k]["line"])
        a, b, c0 = _operands(k)
        ref = _T(c0.extents, c0.strides, ARR[f"k{k}_classical"])
        for run in META[k]["runs"]:
            out = _T(c0.extents, c0.strides, ARR[f"k{k}_L{run['level']}_{run['variant']}"])
            assert oracle.relative_error(out, ref) == run["rel_err"]


def test_oracle_terms_match_reference_table():
    terms = golden_io.terms()
    for level in range(4):
        got = [[list(map(list, s)) for s in t] for t in oracle.strassen_terms(level)]
        assert got == terms[str(level)]


def test_oracle_view_vectors_match_reference():
    meta, arr = golden_io.view_cases()
    for k, cs in enumerate(meta):
        axes = {lab: i for i, lab in enumerate(cs["labels"])}
        rows = [axes[l] for l in cs["rows"]]
        cols = [axes[l] for l in cs["cols"]]
        for q in range(cs["nquads"]):
            rs, cc, rbs, cbs = oracle.view_vectors([cs["ext"][i] for i in rows], [cs["strides"][i] for i in rows],
                                                   [cs["ext"][i] for i in cols], [cs["strides"][i] for i in cols],
                                                   cs["base"], cs["rb"], cs["cb"], cs["level"], q)
            assert np.array_equal(rs, arr[f"c{k}_q{q}_rscat"]), (k, q)
            assert np.array_equal(cc, arr[f"c{k}_q{q}_cscat"]), (k, q)
            assert np.array_equal(rbs, arr[f"c{k}_q{q}_rbs"]), (k, q)
            assert np.array_equal(cbs, arr[f"c{k}_q{q}_cbs"]), (k, q)


def test_reference_unit_goldens_via_oracle():
    # pkg/tests/test_scatter.py:24-29 (A_{d,c,a} view) and :73-77 (partial block)
    rs, cs, rbs, cbs = oracle.view_vectors([4, 2], [16, 8], [8], [1], 0, 8, 4)
    assert rs.tolist() == [0, 16, 32, 48, 8, 24, 40, 56]
    assert rbs.tolist() == [0] and cs.tolist() == list(range(8)) and cbs.tolist() == [1, 1]
    # pad: quadrant 3 of a 7x7 column-major matrix at level 1 (pkg/tests/test_strassen.py:95-99)
    rs, cs, _, _ = oracle.view_vectors([7], [1], [7], [7], 0, 4, 4, level=1, quadrant=3)
    assert rs.tolist() == [4, 5, 6, oracle.PAD]
    assert cs.tolist() == [28, 35, 42, oracle.PAD]


def test_cfg1_golden_summary_consistent():
    g = golden_io.cfg1()
    assert g["leaf_multiplies"] == 7 and len(g["sample_index"]) == 4096
    assert json.dumps(g)  # well-formed
