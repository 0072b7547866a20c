"""n-bundle split host logic with world_size 2 over gloo on CPU (no GPU).

Each rank contracts its J shard with the CPU oracle standing in for the device
kernel (the device path is covered by the -m gpu tests), then the C shards are
all-gathered; the result must equal the unsharded classical contraction
bitwise (the classical nested loop does not depend on the partition).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import paper_1704_03092_b200 as stc
from paper_1704_03092_b200 import shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _operands(spec, seed=5):
    rm = lambda e: tuple(int(np.prod(e[i + 1:])) for i in range(len(e)))
    def t(labels, s):
        e = spec.tensor_extents(labels)
        return stc.DenseTensor(e, rm(e), np.random.default_rng(s).uniform(-1, 1, int(np.prod(e))))
    return t(spec.labels_a, seed), t(spec.labels_b, seed + 1), t(spec.labels_c, seed + 2)


def _oracle_classical(sp, a, b, c, level, variant, **kw):
    oracle.contract_reference(sp, a, b, c)


def _worker(rank, world, port, line, ret):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = stc.parse_benchmark_line(line)
    a, b, c = _operands(spec)
    sh, _ = shard.contract_sharded(spec, a, b, c, 2, "abc", rank, world, contract_fn=_oracle_classical)
    shard.gather_shards(spec, c, rank, world)
    ret[rank] = c.data.copy()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("line,world", [("abcijk abcefg efgijk & a:3;b:2;c:4;i:4;j:3;k:2;e:2;f:3;g:2;", 2),
                                        ("aibj eafb jfie & a:5;b:3;i:6;j:4;e:3;f:2;", 2),
                                        # odd J extents: shards of unequal size (the all-gather pads)
                                        ("aibj eafb jfie & a:4;b:3;i:5;j:3;e:3;f:2;", 2),
                                        ("abcijk abcefg efgijk & a:2;b:3;c:2;i:5;j:7;k:3;e:2;f:3;g:2;", 3)])
def test_nsplit_gloo(line, world):
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), line, ret), nprocs=world, join=True)
    spec = stc.parse_benchmark_line(line)
    a, b, c = _operands(spec)
    oracle.contract_reference(spec, a, b, c)
    for r in range(world):
        assert np.array_equal(ret[r], c.data)


def test_plan_shards_covers_label_exactly():
    spec = stc.parse_benchmark_line("abcijk abcefg efgijk & a:2;b:2;c:2;i:5;j:3;k:8;e:2;f:2;g:2;")
    _, _, c = _operands(spec)
    for world in (1, 2, 3, 4, 8):
        sh = shard.plan_shards(spec, c, world)
        assert sh[0].start == 0 and sh[-1].stop == spec.extents[sh[0].label]
        assert all(x.stop == y.start for x, y in zip(sh, sh[1:]))
        sizes = [s.stop - s.start for s in sh]
        assert max(sizes) - min(sizes) <= 1
    # default label: largest C stride among divisible extents -> i (slowest of J in row-major C)
    assert shard.plan_shards(spec, c, 2)[0].label in "ijk"
    with pytest.raises(ValueError, match="J bundle"):
        shard.plan_shards(spec, c, 2, label="a")


def test_shard_views_address_the_right_elements():
    spec = stc.parse_benchmark_line("aibj eafb jfie & a:3;b:2;i:4;j:6;e:2;f:3;")
    _, b, c = _operands(spec)
    sh = shard.Shard("j", 2, 5)
    cv = shard.shard_tensor(c, spec.labels_c, sh)
    for idx in [(0, 0, 0, 0), (2, 3, 1, 2), (1, 2, 0, 1)]:
        full = (idx[0], idx[1], idx[2], idx[3] + 2)
        assert stc.element_at(cv, idx) == stc.element_at(c, full)
    bv = shard.shard_tensor(b, spec.labels_b, sh)  # B = [j, f, i, e]
    assert stc.element_at(bv, (0, 1, 2, 1)) == stc.element_at(b, (2, 1, 2, 1))


def _grid_worker(rank, world, port, line, gm, gn, ret):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = stc.parse_benchmark_line(line)
    a, b, c = _operands(spec)
    shard.contract_grid(spec, a, b, c, 2, "abc", rank, gm, gn, contract_fn=_oracle_classical)
    shard.gather_blocks(spec, c, rank, gm, gn)
    ret[rank] = c.data.copy()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("gm,gn", [(2, 1), (1, 2), (2, 2)])
def test_grid_split_gloo(gm, gn):
    # the 2-D split over gloo: each rank its (I range, J range) block with the oracle
    # standing in for the device kernel, then the blocks all-gathered (unequal block
    # sizes: extents 5 and 3 split in two)
    line = "abij abef efij & a:5;b:2;i:3;j:4;e:3;f:2;"
    world = gm * gn
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_grid_worker, args=(world, _free_port(), line, gm, gn, ret), nprocs=world, join=True)
    spec = stc.parse_benchmark_line(line)
    a, b, c = _operands(spec)
    oracle.contract_reference(spec, a, b, c)
    for r in range(world):
        assert np.array_equal(ret[r], c.data), r


def test_plan_grid_tiles_c_exactly():
    spec = stc.parse_benchmark_line("abcijk abcefg efgijk & a:3;b:2;c:5;i:5;j:3;k:4;e:2;f:2;g:2;")
    _, _, c = _operands(spec)
    for gm, gn in ((1, 1), (2, 1), (1, 3), (3, 2), (2, 4)):
        blocks = shard.plan_grid(spec, c, gm, gn)
        assert len(blocks) == gm * gn
        seen = np.zeros(c.extents, dtype=int)
        for blk in blocks:
            v = shard.block_tensor(c, spec.labels_c, blk)
            idx = [slice(None)] * len(c.extents)
            for sh in (blk.row, blk.col):
                if sh.label:
                    idx[spec.labels_c.index(sh.label)] = slice(sh.start, sh.stop)
            seen[tuple(idx)] += 1
            assert v.extents == seen[tuple(idx)].shape
        assert (seen == 1).all(), (gm, gn)
        if gm > 1:
            assert blocks[0].row.label in spec.bundle_i
        if gn > 1:
            assert blocks[0].col.label in spec.bundle_j
    with pytest.raises(ValueError, match="I bundle"):
        shard.plan_grid(spec, c, 2, 1, row_label="i")
    with pytest.raises(ValueError, match="extent"):
        shard.plan_grid(spec, c, 7, 1)


@pytest.mark.parametrize("line", ["abcijk abcefg efgijk & a:2;b:2;c:2;i:5;j:3;k:8;e:2;f:2;g:2;",
                                  "aibj eafb jfie & a:4;b:3;i:5;j:3;e:3;f:2;",
                                  "abcij eafbc ifje & a:5;b:7;c:3;i:7;j:9;e:4;f:3;"])
def test_c_abi_shard_planner_matches_plan_shards(line):
    # stc_shard_problem (the C-ABI n-split) and shard.plan_shards / shard_tensor pick the
    # same label, ranges and moved base offsets (host-only: no device needed)
    import ctypes

    from paper_1704_03092_b200 import _lib
    from paper_1704_03092_b200.strassen import Variant, problem_of

    spec = stc.parse_benchmark_line(line)
    a, b, c = _operands(spec)
    prob = problem_of(spec, a, b, c, 2, Variant.ABC)
    for world in (1, 2, 3, 4):
        if max(spec.extents[l] for l in spec.bundle_j) < world:
            continue
        shards = shard.plan_shards(spec, c, world)
        for rank in range(world):
            out = _lib.Problem()
            s0, s1, lab = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
            _lib.check(_lib.lib().stc_shard_problem(ctypes.byref(prob), world, rank, -1, ctypes.byref(out),
                                                    ctypes.byref(s0), ctypes.byref(s1), ctypes.byref(lab)))
            sh = shards[rank]
            assert spec.bundle_j[lab.value] == sh.label and (s0.value, s1.value) == (sh.start, sh.stop)
            want = problem_of(shard.shard_spec(spec, sh), a, shard.shard_tensor(b, spec.labels_b, sh),
                              shard.shard_tensor(c, spec.labels_c, sh), 2, Variant.ABC)
            assert bytes(out) == bytes(want), (world, rank)
