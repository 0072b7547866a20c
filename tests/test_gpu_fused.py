"""GPU parity of the fused TMA kernel (stc_fused.cu) on layouts it accepts.

Each case is a 1024^3 contraction whose views are regular boxes, one per
combination of unit-stride sides (A unit stride in x or k, B unit stride in x
or k), so both raw-view layouts (128-byte swizzled x rows, 64-byte swizzled k
rows) and the fragment permutation are exercised.  Checks:
  * the fused kernel ran (one extra launch: the coordinate table);
  * its C equals the gather kernel's C bitwise (same view order, same DMMA
    k order), for ABC and AB at levels 0..2;
  * normwise relative error <= 1e-12 against the CPU oracle's classical
    contraction (the reference suite's bound; the north star's gate is 1e-10).
"""

import os

import numpy as np
import pytest

import oracle
import paper_1704_03092_b200 as stc

pytestmark = pytest.mark.gpu

TOL = 1e-12
LAYOUTS = {
    # A unit stride in x (b), B unit stride in k (e) -- the BASELINE cfg2 pattern
    "ax_bk": "aibj eafb jfie & a:16;b:64;i:16;j:64;e:64;f:16;",
    # A unit stride in k (f), B unit stride in x (j) -- the 16384^3 bar pattern
    "ak_bx": "abij abef efij & a:16;b:64;i:16;j:64;e:16;f:64;",
    # both unit strides in x
    "ax_bx": "abij eafb efij & a:16;b:64;i:16;j:64;e:16;f:64;",
    # both unit strides in k
    "ak_bk": "abij abef ijef & a:16;b:64;i:16;j:64;e:16;f:64;",
}


def _operands(spec, seed):
    a = stc.make_dense_tensor(spec.tensor_extents(spec.labels_a), "random", seed)
    b = stc.make_dense_tensor(spec.tensor_extents(spec.labels_b), "random", seed + 1)
    c = stc.make_dense_tensor(spec.tensor_extents(spec.labels_c), "random", seed + 2)
    return a.to_device(), b.to_device(), c


def _run(spec, a, b, c0, level, variant, fused):
    # the in-kernel operand sums (pre-summed slots are compared in test_presum_*)
    return _run_env(spec, a, b, c0, level, variant, {"STC_FUSED": "1" if fused else "0", "STC_PRESUM_OPS": "0"})


@pytest.mark.parametrize("name", sorted(LAYOUTS))
def test_fused_matches_gather_bitwise_and_classical(name):
    spec = stc.parse_benchmark_line(LAYOUTS[name])
    a, b, c0 = _operands(spec, 11)
    classical = c0.copy()
    oracle.contract_reference(spec, a.to_host(), b.to_host(), classical)
    for level in (0, 1, 2):
        for variant in ("abc", "ab"):
            cf, stf = _run(spec, a, b, c0, level, variant, True)
            cg, stg = _run(spec, a, b, c0, level, variant, False)
            assert stf.kernel_launches >= stg.kernel_launches, (name, level, variant)  # + the coordinate table on a first call
            assert stf.fast_blocks > 0 and stf.slow_blocks == 0, (name, level, variant)
            assert np.array_equal(cf.data, cg.data), (name, level, variant)
            assert stc.relative_error(cf, classical) <= TOL, (name, level, variant)


def _run_env(spec, a, b, c0, level, variant, env):
    env = {"STC_PRESUM_OPS": "0", **env}  # in-kernel sums unless a test asks for the slots
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        c = c0.to_device()
        st = stc.contract(spec, a, b, c, level, variant)
        return c.to_host(), st
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.mark.parametrize("name", sorted(LAYOUTS))
def test_summing_warpgroup_matches_fragment_sums_bitwise(name):
    # L >= 1: the operand sums are formed once per CTA by the summing warpgroup
    # (STC_PRESUM=3: both sides; 1: the A side, B in the consumers' fragment
    # loads) or all in the fragment loads (0); same view order and roundings,
    # so C must be bitwise equal, with every epilogue mode
    spec = stc.parse_benchmark_line(LAYOUTS[name])
    a, b, c0 = _operands(spec, 61)
    for level in (1, 2):
        for variant in ("abc", "ab"):
            for epi in ({}, {"STC_CRED": "0"}, {"STC_EPI_OFFLOAD": "0"}):
                cf, _ = _run_env(spec, a, b, c0, level, variant, {"STC_PRESUM": "0", **epi})
                for ps in ("1", "3"):
                    cs, _ = _run_env(spec, a, b, c0, level, variant, {"STC_PRESUM": ps, **epi})
                    assert np.array_equal(cs.data, cf.data), (name, level, variant, epi, ps)


@pytest.mark.parametrize("line", [
    LAYOUTS["ax_bk"],
    "abij abef efij & a:24;b:24;i:24;j:24;e:24;f:24;",  # cfg1 (576^3): dense by default
    "abcij eafbc ifje & a:10;b:7;c:13;i:14;j:9;e:18;f:11;",  # irregular, PAD quadrants
])
def test_abc_dense_m_matches_ticketed_bitwise(line):
    # ABC's C updates: straight from the kernel in ticket order, or (many terms in
    # flight per C tile) dense M slots + one accumulate pass in the same order
    # (STC_ABC_DENSE forces either): the same additions, so C must be bitwise equal
    spec = stc.parse_benchmark_line(line)
    a, b, c0 = _operands(spec, 71)
    for level in (1, 2):
        ct, _ = _run_env(spec, a, b, c0, level, "abc", {"STC_ABC_DENSE": "0"})
        cd, _ = _run_env(spec, a, b, c0, level, "abc", {"STC_ABC_DENSE": "1"})
        assert np.array_equal(ct.data, cd.data), (line, level)
        for ps in ("1",):  # pre-summed slots, ticketed (TMA reduce-add where C boxes allow)
            cp, _ = _run_env(spec, a, b, c0, level, "abc", {"STC_ABC_DENSE": "0", "STC_PRESUM_OPS": ps})
            assert np.array_equal(cp.data, cd.data), (line, level, ps)
            for epi in ({"STC_EPI_OFFLOAD": "0"}, {"STC_CRED": "0"}):
                ce, _ = _run_env(spec, a, b, c0, level, "abc", {"STC_ABC_DENSE": "0", "STC_PRESUM_OPS": ps, **epi})
                assert np.array_equal(ce.data, cd.data), (line, level, ps, epi)

        for fused in ("0",):  # the gather kernel takes the same two paths
            cg, _ = _run_env(spec, a, b, c0, level, "abc", {"STC_ABC_DENSE": "1", "STC_FUSED": fused})
            assert np.array_equal(cg.data, cd.data), (line, level)


@pytest.mark.parametrize("line,shape", [
    # I quadrants 64 wide at L2 (m = 256): 64 x 256 tiles; J quadrants 64 wide: 256 x 64
    ("abij abef efij & a:16;b:16;i:32;j:64;e:32;f:16;", 1),
    ("abij abef efij & a:64;b:32;i:16;j:16;e:32;f:16;", 2),
    ("aibj eafb jfie & a:16;b:16;i:16;j:128;e:16;f:32;", 1),
    # cfg1 (576^3) L1: 64 x 128 tiles on 32 x 32 warp tiles (the items do not fill the SMs)
    ("abij abef efij & a:24;b:24;i:24;j:24;e:24;f:24;", 3),
    # J quadrants of 150 (L2): 128 x 64 tiles pad them to 192 instead of 256 (dense-M plans)
    ("abij abef efij & a:20;b:40;i:24;j:25;e:16;f:32;", 4),
])
def test_tile_shapes_match_square_tiles_bitwise(line, shape):
    # the 64 x 256 / 256 x 64 CTA tiles (dense-M launches with the summing warpgroup) give
    # every M element the same k order and sums as the 128 x 128 tiles (STC_TSHAPE=0)
    spec = stc.parse_benchmark_line(line)
    a, b, c0 = _operands(spec, 81)
    classical = c0.copy()
    oracle.contract_reference(spec, a.to_host(), b.to_host(), classical)
    if shape == 3:  # (or 128 x 64 on the same 32 x 32 warp tiles: the same padded area)
        assert stc.describe_plan(spec, a, b, c0, 1, "abc")["tshape"] in (3, 4)
    if shape == 4:
        assert stc.describe_plan(spec, a, b, c0, 2, "ab")["tshape"] == 4
    for level, variant in ((2, "ab"), (2, "abc"), (1, "ab"), (1, "abc")):
        cs, ss = _run_env(spec, a, b, c0, level, variant, {})
        cq, sq = _run_env(spec, a, b, c0, level, variant, {"STC_TSHAPE": "0"})
        assert np.array_equal(cs.data, cq.data), (line, level, variant)
        assert stc.relative_error(cs, classical) <= TOL
        if level == 2 and shape in (1, 2):  # the shaped launch has half the padded work items
            assert ss.work_items < sq.work_items, (ss.work_items, sq.work_items)
        # the same shapes on pre-summed slots (one view per side): bitwise the same again
        cp, sp_ = _run_env(spec, a, b, c0, level, variant, {"STC_PRESUM_OPS": "1"})
        assert np.array_equal(cp.data, cq.data), (line, level, variant)
        if level == 2 and shape in (1, 2):
            assert sp_.work_items == ss.work_items, (sp_.work_items, ss.work_items)


@pytest.mark.parametrize("line", [
    "abij abef efij & a:16;b:16;i:32;j:64;e:32;f:16;",   # m = 256: 64 x 256 tiles, A slots only
    "abij abef efij & a:64;b:32;i:16;j:16;e:32;f:16;",   # n = 256: 256 x 64 tiles, B slots only
    "aibj eafb jfie & a:16;b:16;i:16;j:128;e:16;f:32;",  # m = 256, permuted layouts
])
def test_one_sided_presum_matches_bitwise(line):
    # one side's sums from k_presum slots, the other's formed in the kernel: every M
    # element sees the same sums in the same order -> bitwise the in-kernel / both-sided C
    spec = stc.parse_benchmark_line(line)
    a, b, c0 = _operands(spec, 85)
    classical = c0.copy()
    oracle.contract_reference(spec, a.to_host(), b.to_host(), classical)
    for level, variant in ((2, "abc"), (2, "ab"), (1, "abc")):
        ref, _ = _run_env(spec, a, b, c0, level, variant, {"STC_PRESUM_OPS": "0", "STC_PRESUM_SIDES": "0"})
        assert stc.relative_error(ref, classical) <= TOL
        for sides in ("1", "2", "3"):
            env = {"STC_PRESUM_SIDES": sides}
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            try:
                info = stc.describe_plan(spec, a, b, c0, level, variant)
            finally:
                for k, v in old.items():
                    os.environ.pop(k) if v is None else os.environ.__setitem__(k, v)
            cs, st = _run_env(spec, a, b, c0, level, variant, env)
            assert np.array_equal(cs.data, ref.data), (line, level, variant, sides, info)
            assert st.leaf_multiplies == 7 ** level
    # the default plan of the 64-wide case at L2 takes the one-sided slots
    assert stc.describe_plan(spec, a, b, c0, 2, "abc")["presum_sides"] in (1, 2)


def test_fused_matches_oracle_strassen():
    # the oracle's own L2 ABC Strassen on the same inputs (different summation
    # order inside the leaf GEMMs, so compared in norm)
    spec = stc.parse_benchmark_line(LAYOUTS["ax_bk"])
    a, b, c0 = _operands(spec, 21)
    ref = c0.copy()
    oracle.contract(spec, a.to_host(), b.to_host(), ref, 2, "abc")
    cf, st = _run(spec, a, b, c0, 2, "abc", True)
    assert st.leaf_multiplies == 49
    assert stc.relative_error(cf, ref) <= TOL


def test_forced_slow_uses_the_gather_kernel():
    # force_slow (the reference's per-element packing) always takes the gather kernel
    spec = stc.parse_benchmark_line(LAYOUTS["ak_bx"])
    a, b, c0 = _operands(spec, 32)
    c = c0.to_device()
    st = stc.contract(spec, a, b, c, 1, "abc", force_slow=True)
    assert st.fast_blocks == 0 and st.slow_blocks > 0


def test_epilogue_modes_are_bitwise_identical():
    # C updates: inline or by the producer warpgroup's spare warps (STC_EPI_OFFLOAD),
    # with TMA reduce-add (default when the C targets are regular) or load/add/store
    # (STC_CRED=0); every combination must give the same C
    spec = stc.parse_benchmark_line(LAYOUTS["ak_bx"])
    a, b, c0 = _operands(spec, 41)
    outs = {}
    for cred in ("1", "0"):
        for off in ("0", "1"):
            os.environ["STC_CRED"], os.environ["STC_EPI_OFFLOAD"] = cred, off
            try:
                outs[cred, off] = [_run(spec, a, b, c0, level, "abc", True)[0].data for level in (1, 2)]
            finally:
                del os.environ["STC_CRED"], os.environ["STC_EPI_OFFLOAD"]
    ref = outs["1", "1"]
    for key, got in outs.items():
        for level in range(2):
            assert np.array_equal(got[level], ref[level]), (key, level + 1)


@pytest.mark.parametrize("line", [
    # the BASELINE irregular stress pattern, shrunk: odd extents, PAD quadrants
    "abcij eafbc ifje & a:10;b:7;c:13;i:14;j:9;e:18;f:11;",
    # permuted regular-looking layout whose tiles are not boxes (extent 24)
    "abij abef efij & a:24;b:24;i:24;j:24;e:24;f:24;",
])
def test_repacked_operands_match_gather_bitwise(line):
    # irregular views: A and B are repacked into dense quadrant blocks and the
    # fused kernel runs on those (one extra pack + pool launch per operand);
    # results must equal the gather kernel's bitwise, and the classical result
    spec = stc.parse_benchmark_line(line)
    a, b, c0 = _operands(spec, 51)
    classical = c0.copy()
    oracle.contract_reference(spec, a.to_host(), b.to_host(), classical)
    for level in (0, 1, 2):
        for variant in ("abc", "ab"):
            cf, stf = _run(spec, a, b, c0, level, variant, True)
            cg, stg = _run(spec, a, b, c0, level, variant, False)
            # the two repacking launches (the pool / coordinate set-up is restored from the
            # plan's snapshot after the first call)
            assert stf.kernel_launches >= stg.kernel_launches + 2, (level, variant)
            assert np.array_equal(cf.data, cg.data), (level, variant)
            assert stc.relative_error(cf, classical) <= TOL, (level, variant)


def test_host_c_upload_overlap_matches():
    # STC_C_OVERLAP=1: a host C is uploaded on a side stream while the kernel's
    # main loop runs; the kernels wait on the device flag (stc_set_c_ready)
    spec = stc.parse_benchmark_line(LAYOUTS["ax_bk"])
    a = stc.make_dense_tensor(spec.tensor_extents(spec.labels_a), "random", 61)
    b = stc.make_dense_tensor(spec.tensor_extents(spec.labels_b), "random", 62)
    c0 = stc.make_dense_tensor(spec.tensor_extents(spec.labels_c), "random", 63)
    outs = []
    os.environ["STC_HOST_PIPELINE"] = "0"  # the staged path (host operands uploaded whole)
    for flag in ("0", "1"):
        os.environ["STC_C_OVERLAP"] = flag
        try:
            for variant in ("abc", "ab", "naive"):
                c = c0.copy()
                stc.contract(spec, a, b, c, 2, variant)
                outs.append(c.data.copy())
        finally:
            del os.environ["STC_C_OVERLAP"]
    del os.environ["STC_HOST_PIPELINE"]
    for i in range(3):
        assert np.array_equal(outs[i], outs[i + 3])


@pytest.mark.parametrize("name", ["ax_bk", "ak_bx"])
def test_integer_data_exact_on_every_path(name):
    # integer-valued inputs: every product and partial sum is exact, so C must equal the
    # classical result bitwise on the fused path (direct and repacked operands, TMA-reduce
    # and load/add/store epilogues, inline and offloaded) for ABC, AB and Naive at L0..L2
    spec = stc.parse_benchmark_line(LAYOUTS[name])

    def ints(labels, seed):
        e = spec.tensor_extents(labels)
        return stc.DenseTensor(e, tuple(int(np.prod(e[i + 1:])) for i in range(len(e))),
                               np.random.default_rng(seed).integers(-8, 9, int(np.prod(e))).astype(np.float64))

    a, b, c0 = ints(spec.labels_a, 71), ints(spec.labels_b, 72), ints(spec.labels_c, 73)
    ref = c0.copy()
    oracle.contract_reference(spec, a, b, ref, threads=8)
    ad, bd = a.to_device(), b.to_device()
    envs = [{}, {"STC_CRED": "0"}, {"STC_EPI_OFFLOAD": "0"}, {"STC_PACK": "1", "STC_FUSED": "1"}]
    for env in envs:
        os.environ.update(env)
        try:
            for level in (0, 1, 2):
                for variant in ("abc", "ab", "naive"):
                    c = c0.to_device()
                    stc.contract(spec, ad, bd, c, level, variant)
                    assert np.array_equal(c.to_host().data, ref.data), (env, level, variant)
        finally:
            for k in env:
                del os.environ[k]


@pytest.mark.parametrize("offset", [0, 1, 2])
def test_strided_torch_views(offset):
    # operands as strided torch views (permuted strides, storage offsets): the fused path
    # needs 16-byte aligned map bases, so odd offsets take the repacked path; results must
    # match a classical einsum on the same views
    import torch

    spec = stc.parse_benchmark_line(LAYOUTS["ax_bk"])
    g = torch.Generator(device="cuda").manual_seed(81)

    def view(labels):
        e = spec.tensor_extents(labels)
        n = int(np.prod(e))
        flat = torch.rand(n + 8, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        return torch.as_strided(flat, e, tuple(int(np.prod(e[i + 1:])) for i in range(len(e))), offset)

    a, b, c = view(spec.labels_a), view(spec.labels_b), view(spec.labels_c)
    ref = c + torch.einsum(f"{spec.labels_a},{spec.labels_b}->{spec.labels_c}", a, b)
    for level, variant in ((2, "abc"), (1, "ab")):
        cc = c.clone()
        stc.contract(spec, a, b, cc, level, variant)
        assert (torch.linalg.vector_norm(cc - ref) / torch.linalg.vector_norm(ref)).item() <= TOL


def test_random_contractions_fuzz():
    # tools/fuzz_gpu.py: random labels / extents / permuted layouts / storage offsets, all
    # variants and levels, against a classical einsum (a fixed-seed slice of the sweep)
    import importlib.util
    import pathlib

    path = pathlib.Path(__file__).resolve().parents[1] / "tools" / "fuzz_gpu.py"
    spec = importlib.util.spec_from_file_location("fuzz_gpu", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    assert mod.main(24, 7) == 0


@pytest.mark.parametrize("name", sorted(LAYOUTS))
def test_presummed_operands_match_in_kernel_sums_bitwise(name):
    # k_presum forms every term's operand sums once per element position (same view order
    # and roundings as the in-SM sums), the fused kernel then reads one slot per side:
    # C must be bitwise equal to the in-kernel sums, for every C-update path
    spec = stc.parse_benchmark_line(LAYOUTS[name])
    a, b, c0 = _operands(spec, 67)
    for level in (1, 2):
        for variant in ("abc", "ab"):
            for epi in ({}, {"STC_ABC_DENSE": "1"}, {"STC_CRED": "0"}):
                ck, _ = _run_env(spec, a, b, c0, level, variant, {"STC_PRESUM_OPS": "0", **epi})
                cp, st = _run_env(spec, a, b, c0, level, variant, {"STC_PRESUM_OPS": "1", **epi})
                assert np.array_equal(cp.data, ck.data), (name, level, variant, epi)
                assert st.fast_blocks > 0 and st.leaf_multiplies == 7 ** level


@pytest.mark.parametrize("line", [
    "abcij eafbc ifje & a:10;b:7;c:13;i:14;j:9;e:18;f:11;",  # irregular, PAD quadrants
    "abcijk abcefg efgijk & a:4;b:8;c:8;i:4;j:8;k:8;e:4;f:8;g:8;",  # cfg5 pattern: 8-wide C runs at L2
])
def test_presummed_irregular_layouts_match_oracle(line):
    spec = stc.parse_benchmark_line(line)
    a, b, c0 = _operands(spec, 73)
    classical = c0.copy()
    oracle.contract_reference(spec, a.to_host(), b.to_host(), classical)
    for level in (1, 2):
        for variant in ("abc", "ab", "naive"):
            cp, _ = _run_env(spec, a, b, c0, level, variant, {"STC_PRESUM_OPS": "1"})
            ck, _ = _run_env(spec, a, b, c0, level, variant, {"STC_PRESUM_OPS": "0"})
            assert np.array_equal(cp.data, ck.data), (line, level, variant)
            assert stc.relative_error(cp, classical) <= TOL, (line, level, variant)


def _run_env_deep(spec, a, b, c0, variant, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        c = c0.to_device()
        st = stc.contract(spec, a, b, c, 3, variant, allow_deep=True)
        return c.to_host(), st
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.mark.parametrize("line", [
    LAYOUTS["ax_bk"], LAYOUTS["ak_bx"],
    "abcij eafbc ifje & a:10;b:7;c:13;i:14;j:9;e:18;f:11;",  # irregular, PAD quadrants at L3
])
def test_level_three_presummed_slots_match_gather_kernel_bitwise(line):
    # L3 (allow_deep): the 343 terms' operand sums (up to 8 views a side) come from k_presum<3>
    # slots and run on the fused one-view kernel; bitwise equal to the gather kernel forming
    # the same sums in its producers (STC_PRESUM_OPS=0), every variant, and to the oracle
    spec = stc.parse_benchmark_line(line)
    a, b, c0 = _operands(spec, 83)
    classical = c0.copy()
    oracle.contract_reference(spec, a.to_host(), b.to_host(), classical)
    for variant in ("abc", "ab", "naive"):
        cp, st = _run_env_deep(spec, a, b, c0, variant, {})
        assert st.leaf_multiplies == 343 and st.fast_blocks > 0, (line, variant, st)
        assert stc.relative_error(cp, classical) <= TOL, (line, variant)
        if variant != "naive":
            ck, _ = _run_env_deep(spec, a, b, c0, variant, {"STC_PRESUM_OPS": "0"})
            assert np.array_equal(cp.data, ck.data), (line, variant)
    plan = stc.describe_plan(spec, a, b, c0, 3, "abc")
    assert plan["presum"] == 1 and plan["terms"] == 343, plan


@pytest.mark.parametrize("line,level", [
    ("abcij eafbc ifje & a:50;b:7;c:13;i:70;j:45;e:90;f:33;", 0),  # cfg4 L0: the consumers' scatter epilogue
    ("aibj eafb jfie & a:32;b:64;i:32;j:64;e:32;f:32;", 2),         # L2 ABC, TMA reduce-add epilogue
])
def test_repeated_runs_bitwise_stable(line, level):
    # regression guard for the TMA-refill race (a stage refilled while
    # fragment loads were in flight gave wrong 64-row blocks about 1 run in 4): the same
    # contraction repeated must give the same bits every time, on both C-update paths
    spec = stc.parse_benchmark_line(line)
    a, b, c0 = _operands(spec, 79)
    for ps in ("0", "1"):
        first, _ = _run_env(spec, a, b, c0, level, "abc", {"STC_PRESUM_OPS": ps})
        for _ in range(12):
            again, _ = _run_env(spec, a, b, c0, level, "abc", {"STC_PRESUM_OPS": ps})
            assert np.array_equal(again.data, first.data), (line, level, ps)


def test_eight_wide_c_boxes_match_dense_m_bitwise():
    # cfg5 pattern, row-major: at L2 the C quadrants hold 8-wide runs of the unit-stride
    # label k (a quadrant split of it), so the TMA reduce-add boxes have 64-byte rows
    # (GemmArgs::cred8, 64B swizzle): bitwise equal to the dense-M accumulate path
    spec = stc.parse_benchmark_line("abcijk abcefg efgijk & a:4;b:8;c:32;i:4;j:8;k:32;e:4;f:8;g:32;")

    def rm_tensor(labels, seed):
        e = spec.tensor_extents(labels)
        st = tuple(int(np.prod(e[i + 1:])) for i in range(len(e)))
        return stc.DenseTensor(e, st, np.random.default_rng(seed).uniform(-1, 1, int(np.prod(e))))

    a, b, c0 = rm_tensor(spec.labels_a, 81), rm_tensor(spec.labels_b, 82), rm_tensor(spec.labels_c, 83)
    info = stc.describe_plan(spec, a, b, c0, 2, "abc")
    assert info["c_boxes"] == 1 and info["presum"] == 1, info
    classical = c0.copy()
    oracle.contract_reference(spec, a, b, classical)
    cd, _ = _run_env(spec, a, b, c0, 2, "abc", {"STC_ABC_DENSE": "1", "STC_PRESUM_OPS": "1"})
    assert stc.relative_error(cd, classical) <= TOL
    for env in ({"STC_ABC_DENSE": "0", "STC_PRESUM_OPS": "1"},
                {"STC_ABC_DENSE": "0", "STC_PRESUM_OPS": "1", "STC_EPI_OFFLOAD": "0"},
                {"STC_ABC_DENSE": "0", "STC_PRESUM_OPS": "0"},
                {"STC_ABC_DENSE": "0", "STC_PRESUM_OPS": "0", "STC_CRED": "0"}):
        ct, _ = _run_env(spec, a, b, c0, 2, "abc", env)
        assert np.array_equal(ct.data, cd.data), env


@pytest.mark.parametrize("line", [
    "abij abef efij & a:24;b:24;i:24;j:24;e:24;f:24;",   # cfg1 geometry (576^3)
    "aibj eafb jfie & a:16;b:32;i:16;j:32;e:32;f:16;",   # cfg2's permuted layouts, 512^3
])
def test_tile_config_params_bitwise(line):
    # contract(params=TileConfig(...)): every CTA tile shape and ring depth gives the C of
    # the planner's choice bitwise (the tile config only reschedules the same DMMA k-steps)
    spec = stc.parse_benchmark_line(line)
    a, b, c0 = _operands(spec, 97)
    classical = c0.copy()
    oracle.contract_reference(spec, a.to_host(), b.to_host(), classical)
    for level, variant in ((1, "abc"), (2, "ab"), (2, "abc")):
        base = c0.to_device()
        stc.contract(spec, a, b, base, level, variant)
        base = base.to_host()
        assert stc.relative_error(base, classical) <= TOL
        configs = [stc.TileConfig(cta_tile=t) for t in sorted(stc.CTA_TILES)]
        configs += [stc.TileConfig(stages=s) for s in (2, 3, 5)]
        configs += [stc.TileConfig(cta_tile=(64, 128), stages=2)]
        for cfg in configs:
            c = c0.to_device()
            stc.contract(spec, a, b, c, level, variant, params=cfg)
            if cfg.cta_tile is not None:
                assert stc.describe_plan(spec, a, b, c0, level, variant, params=cfg)["tshape"] == \
                    stc.CTA_TILES[cfg.cta_tile]
            assert np.array_equal(c.to_host().data, base.data), (line, level, variant, cfg)


@pytest.mark.parametrize("line", [
    # a short I / J with a very long P: the repacked operands' [k][x] blocks have 262144
    # rows (k_pack_views' row blocks once overflowed grid.y and the error was dropped)
    "ij ie ej & i:16;j:64;e:262144;",
    "di edbc ecbi & d:16;i:64;e:128;b:32;c:64;",
])
def test_long_k_repacked_operands(line):
    import torch

    spec = stc.parse_benchmark_line(line)
    gen = torch.Generator(device="cuda").manual_seed(5)

    def dev(labels):
        e = spec.tensor_extents(labels)
        return (torch.rand(e, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1).contiguous()

    a, b, c0 = dev(spec.labels_a), dev(spec.labels_b), dev(spec.labels_c)
    ref = c0 + torch.einsum(f"{spec.labels_a},{spec.labels_b}->{spec.labels_c}", a, b)
    out = {}
    for fused in ("1", "0"):
        os.environ["STC_FUSED"] = fused
        try:
            for level in (0, 1):
                c = c0.clone()
                st = stc.contract(spec, a, b, c, level, "abc")
                assert st.leaf_multiplies == 7 ** level
                err = (torch.linalg.vector_norm(c - ref) / torch.linalg.vector_norm(ref)).item()
                assert err <= TOL, (line, fused, level, err)
                out[fused, level] = c
        finally:
            os.environ.pop("STC_FUSED", None)
    assert torch.equal(out["1", 0], out["0", 0])  # repacked fused kernel == gather kernel, bitwise
