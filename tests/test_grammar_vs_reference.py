"""The benchmark-line grammar against the reference's own parser (CPU; skipped where
/root/reference is absent, e.g. on the GPU box).

Random well-formed and malformed lines go through both ``parse_benchmark_line``s
(reference: pkg/src/strassen_tc/tensor.py:196-228, ContractionSpec checks :150-165):
the same spec, or the same exception type and message.
"""

from __future__ import annotations

import pathlib
import random
import sys

import pytest

import paper_1704_03092_b200 as stc

REF_SRC = pathlib.Path("/root/reference/pkg/src")


@pytest.fixture(scope="module")
def ref_tensor():
    if not (REF_SRC / "strassen_tc" / "tensor.py").exists():
        pytest.skip("reference sources not present")
    sys.path.insert(0, str(REF_SRC))
    try:
        import strassen_tc.tensor as ref
    except Exception as exc:  # its package __init__ pulls numba
        pytest.skip(f"reference not importable: {exc}")
    finally:
        sys.path.remove(str(REF_SRC))
    return ref


def _outcome(parse, line):
    try:
        s = parse(line)
    except Exception as exc:  # noqa: BLE001 -- the comparison is the point
        return type(exc).__name__, str(exc)
    return "ok", s.labels_c, s.labels_a, s.labels_b, s.extents, s.bundle_i, s.bundle_j, s.bundle_p


def _lines(rng, count):
    noise = "abcdeA1 :;&_+-0123"
    for t in range(count):
        if t % 2:
            yield "".join(rng.choice(noise) for _ in range(rng.randint(0, 25)))
            continue
        groups = ["".join(rng.sample("abcde", rng.randint(1, 3))) for _ in range(3)]
        if rng.random() < 0.2:
            groups[0] += groups[0][0]
        ext = ";".join(f"{lab}:{rng.choice([0, 1, 2, 3, 'x', ' 4', '+2'])}"
                       for lab in rng.sample("abcdez", rng.randint(2, 6)))
        yield " ".join(groups) + " & " + ext + rng.choice(["", ";"])


def test_parser_matches_reference_on_random_lines(ref_tensor):
    rng = random.Random(1704)
    mismatches = [line for line in _lines(rng, 20000)
                  if _outcome(ref_tensor.parse_benchmark_line, line) != _outcome(stc.parse_benchmark_line, line)]
    assert not mismatches, mismatches[:5]
