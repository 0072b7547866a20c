"""GPU: the tiny-shape cases of the reference's driver tests (pkg/tests/test_driver.py:43-104,
165-183) on the DMMA kernel: 1 x 1 x 1, 2 x 2, identity B, a singleton fused primitive bitwise
equal to the dense GEMM, force_slow bitwise neutral, repeated runs bitwise stable."""

import numpy as np
import pytest

import paper_1704_03092_b200 as stc

pytestmark = pytest.mark.gpu
SMALL = stc.BlockingParams(mc=8, nc=8, kc=4, mr=4, nr=2, kr=2)


def cm(x):
    import torch

    return torch.from_numpy(np.asfortranarray(np.asarray(x, dtype=np.float64))).cuda()


def dense_problem(m, n, k, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, (m, k)), rng.uniform(-1, 1, (k, n)), rng.uniform(-1, 1, (m, n))


def test_scalar_fma_and_two_by_two_identity():
    c = cm(np.full((1, 1), 1.0))
    st = stc.run_gemm_dense(c, cm(np.full((1, 1), 3.0)), cm(np.full((1, 1), 5.0)), SMALL)
    assert c.item() == 16.0 and st.leaf_multiplies == 1
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    c = cm(np.zeros((2, 2)))
    stc.run_gemm_dense(c, cm(a), cm(np.eye(2)), SMALL)
    assert np.array_equal(c.cpu().numpy(), a)


@pytest.mark.parametrize("n", [6, 129, 257])
def test_identity_b_accumulates_a_exactly(n):
    a, _, _ = dense_problem(n, n, n, n)
    c = cm(np.zeros((n, n)))
    stc.run_gemm_dense(c, cm(a), cm(np.eye(n)), SMALL)
    assert np.array_equal(c.cpu().numpy(), a)  # a * 1 + zeros: exact in any summation order


@pytest.mark.parametrize("shape", [(13, 17, 11), (1, 300, 7), (300, 1, 7), (5, 5, 1), (129, 130, 131)])
def test_random_gemm_matches_numpy(shape):
    m, n, k = shape
    a, b, c = dense_problem(m, n, k, 3)
    tc = cm(c)
    stc.run_gemm_dense(tc, cm(a), cm(b), SMALL)
    ref = c + a @ b
    assert np.linalg.norm(tc.cpu().numpy() - ref) / np.linalg.norm(ref) < 1e-13


def _view(t, rb, cb):
    return stc.matrix_view(stc.DenseTensor.from_torch(t), rb, cb)


def test_singleton_fused_equals_dense_gemm_bitwise_and_force_slow_neutral():
    import torch

    a, b, c = dense_problem(12, 10, 6, 7)
    ta, tb = cm(a), cm(b)
    outs = []
    for force_slow in (False, True):
        tc = cm(c)
        prim = stc.FusedPrimitive(stc.OperandTermSide([_view(ta, SMALL.mr, SMALL.kr)], [1]),
                                  stc.OperandTermSide([_view(tb, SMALL.kr, SMALL.nr)], [1]),
                                  stc.OperandTermSide([_view(tc, SMALL.mr, SMALL.nr)], [1]))
        stc.run_fused(prim, SMALL, force_slow=force_slow)
        outs.append(tc)
    t2 = cm(c)
    stc.run_gemm_dense(t2, ta, tb, SMALL)
    assert torch.equal(outs[0], t2) and torch.equal(outs[1], t2)
    t3 = cm(c)
    stc.run_gemm_dense(t3, ta, tb, SMALL, threads=3)  # threads: accepted, ignored
    assert torch.equal(t3, t2)


def test_total_flops_counts_executed_tiles():
    a, b, c = dense_problem(4, 4, 4, 12)
    st = stc.run_gemm_dense(cm(c), cm(a), cm(b), SMALL)
    # GPU tiles replace the mr x nr register blocks: the count is a whole number of padded CTA tiles
    assert st.total_flops >= 2 * 4 * 4 * 4 and st.leaf_multiplies == 1
