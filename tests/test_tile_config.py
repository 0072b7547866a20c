"""TileConfig -- the GPU tile config that replaces the reference's BlockingParams
(kernels.py:34-56) as contract()'s ``params``: validation, its
stc_problem.tiling code, and the plans it produces (stc_plan_describe, host-only)."""

import numpy as np
import pytest

import paper_1704_03092_b200 as stc

CFG1 = "abij abef efij & a:24;b:24;i:24;j:24;e:24;f:24;"
CFG2_SMALL = "aibj eafb jfie & a:16;b:32;i:16;j:32;e:32;f:16;"


def _operands(line):
    spec = stc.parse_benchmark_line(line)

    def t(labels):
        e = spec.tensor_extents(labels)
        return stc.make_dense_tensor(e)

    return spec, t(spec.labels_a), t(spec.labels_b), t(spec.labels_c)


def test_tile_config_validation_and_code():
    assert stc.TileConfig().code == 0
    assert stc.TileConfig(cta_tile=(128, 128)).code == 1
    assert stc.TileConfig(cta_tile=[64, 128], stages=4).code == 4 | (4 << 4)
    with pytest.raises(ValueError, match="cta_tile"):
        stc.TileConfig(cta_tile=(96, 96))
    with pytest.raises(ValueError, match="stages"):
        stc.TileConfig(stages=1)
    with pytest.raises(ValueError, match="stages"):
        stc.TileConfig(stages=9)


def test_params_type_is_checked():
    spec, a, b, c = _operands(CFG1)
    with pytest.raises(TypeError, match="TileConfig"):
        stc.describe_plan(spec, a, b, c, 1, stc.Variant.ABC, params=object())


@pytest.mark.parametrize("tile", sorted(stc.CTA_TILES))
def test_requested_shape_is_planned(tile):
    spec, a, b, c = _operands(CFG1)
    info = stc.describe_plan(spec, a, b, c, 1, stc.Variant.AB, params=stc.TileConfig(cta_tile=tile))
    assert info["tshape"] == stc.CTA_TILES[tile], info
    assert info["mq_pad"] % tile[0] == 0 and info["nq_pad"] % tile[1] == 0, info


def test_blocking_params_leave_the_planner_in_charge():
    spec, a, b, c = _operands(CFG1)
    default = stc.describe_plan(spec, a, b, c, 1, stc.Variant.ABC)
    ref_blocking = stc.describe_plan(spec, a, b, c, 1, stc.Variant.ABC, params=stc.BlockingParams(mc=48, nc=96))
    assert default == ref_blocking


def test_shape_needs_a_strassen_level_and_not_naive():
    spec, a, b, c = _operands(CFG2_SMALL)
    with pytest.raises(ValueError, match="tile shape"):
        stc.describe_plan(spec, a, b, c, 0, stc.Variant.ABC, params=stc.TileConfig(cta_tile=(64, 128)))
    with pytest.raises(ValueError, match="tile shape"):
        stc.describe_plan(spec, a, b, c, 1, stc.Variant.NAIVE, params=stc.TileConfig(cta_tile=(64, 256)))
    # the default 128 x 128 tile is always available
    info = stc.describe_plan(spec, a, b, c, 0, stc.Variant.ABC, params=stc.TileConfig(cta_tile=(128, 128)))
    assert info["tshape"] == 0
