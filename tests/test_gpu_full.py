"""GPU parity at full BASELINE sizes against the REFERENCE's own outputs.

tests/golden/full.json holds the reference contract()'s results for cfg2
(4096^3 permuted layouts, L1 / L2 ABC) and cfg4 (the irregular 4550 x 3150 x 2970
stress config, AB and Naive at L1 / L2), computed on the reference's CPU path
(tests/golden/make_golden.py --full) and summarised by the Frobenius norm, the
sum and 4096 sampled entries.  Inputs are rebuilt here with the same seeds.
Tolerance 1e-12 normwise (the reference suite's bound; the north star's gate is
1e-10): the leaf GEMMs sum in a different order from the reference's micro-kernel.
"""

import json
import pathlib

import numpy as np
import pytest

import paper_1704_03092_b200 as stc

pytestmark = pytest.mark.gpu

TOL = 1e-12
FULL = json.loads((pathlib.Path(__file__).resolve().parent / "golden" / "full.json").read_text())


def _rm(ext):
    return tuple(int(np.prod(ext[i + 1:])) for i in range(len(ext)))


def _tensor(spec, labels, seed, fill, device):
    ext = spec.tensor_extents(labels)
    n = int(np.prod(ext))
    rng = np.random.default_rng(seed)
    data = rng.uniform(-1.0, 1.0, n) if fill == "uniform" else rng.standard_normal(n)
    return stc.DenseTensor(ext, _rm(ext), data).to_device(device)


@pytest.mark.parametrize("case", FULL, ids=[f"{c['name']}-L{c['level']}-{c['variant']}" for c in FULL])
def test_full_size_against_reference_output(case):
    import torch

    dev = torch.device("cuda", 0)
    spec = stc.parse_benchmark_line(case["line"])
    a = _tensor(spec, spec.labels_a, case["seed_a"], case["fill"], dev)
    b = _tensor(spec, spec.labels_b, case["seed_b"], case["fill"], dev)
    ext_c = spec.tensor_extents(spec.labels_c)
    c = stc.DenseTensor(ext_c, _rm(ext_c), torch.zeros(int(np.prod(ext_c)), dtype=torch.float64, device=dev))
    st = stc.contract(spec, a, b, c, case["level"], case["variant"])
    assert st.leaf_multiplies == case["leaf_multiplies"] == 7 ** case["level"]
    flat = c.data
    frob = float(torch.linalg.vector_norm(flat))
    assert abs(frob - case["frob"]) <= TOL * case["frob"]
    idx = torch.tensor(case["sample_index"], device=dev)
    got = flat[idx].cpu().numpy()
    ref = np.array(case["sample_value"])
    assert np.linalg.norm(got - ref) <= TOL * np.linalg.norm(ref)
