"""Multi-GPU split paths (north-star subsystem 5) on the
CUDA path, checked against the CPU oracle through the split.

* n-split and 2-D grid on one GPU: every rank's part of C is contracted by the
  B200 kernels (ranks one after another on this GPU -- the shards share no data
  and need no collective), and the same shards are contracted by the oracle's
  restatement of the reference (oracle.contract, the reference's own Strassen
  partition of each shard): shard by shard within 1e-12, and the assembled C
  against the classical oracle within 1e-12.  Odd extents: shards of unequal size.
* two ranks over NCCL (skipped with fewer than 2 GPUs): each rank its shard on
  its own GPU, then shard.gather_shards (NCCL all-gather), against the oracle.
"""

import os
import socket

import numpy as np
import pytest

import oracle
import paper_1704_03092_b200 as stc
from paper_1704_03092_b200 import shard

pytestmark = pytest.mark.gpu
TOL = 1e-12
LINE = "abcijk abcefg efgijk & a:6;b:5;c:7;i:5;j:6;k:7;e:5;f:6;g:7;"


def _rm(e):
    return tuple(int(np.prod(e[i + 1:])) for i in range(len(e)))


def _host(spec, seed=23):
    def t(labels, s):
        e = spec.tensor_extents(labels)
        return stc.DenseTensor(e, _rm(e), np.random.default_rng(s).uniform(-1, 1, int(np.prod(e))))
    return t(spec.labels_a, seed), t(spec.labels_b, seed + 1), t(spec.labels_c, seed + 2)


def _oracle_fn(level, variant):
    def fn(sp, a, b, c, lv, var, **kw):
        oracle.contract(sp, a, b, c, level, variant, threads=oracle.max_threads())
    return fn


def _classical(spec, a, b, c):
    ref = c.copy()
    oracle.contract_reference(spec, a, b, ref, threads=oracle.max_threads())
    return ref


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("level,variant", [(1, "abc"), (2, "abc"), (2, "ab"), (2, "naive")])
def test_nsplit_cuda_against_oracle(world, level, variant):
    spec = stc.parse_benchmark_line(LINE)
    a, b, c0 = _host(spec)
    A, B = a.to_device(), b.to_device()
    C = c0.to_device()
    ref = c0.copy()
    for rank in range(world):
        sh, st = shard.contract_sharded(spec, A, B, C, level, variant, rank, world)
        assert st.leaf_multiplies == 7 ** level
        shard.contract_sharded(spec, a, b, ref, level, variant, rank, world, contract_fn=_oracle_fn(level, variant))
        got = stc.DenseTensor(c0.extents, c0.strides, C.data.cpu().numpy())
        # this rank's shard: GPU vs the reference algorithm on the same shard
        err = oracle.relative_error(shard.shard_tensor(got, spec.labels_c, sh), shard.shard_tensor(ref, spec.labels_c, sh))
        assert err <= TOL, (rank, err)
    got = stc.DenseTensor(c0.extents, c0.strides, C.data.cpu().numpy())
    assert oracle.relative_error(got, _classical(spec, a, b, c0)) <= TOL


@pytest.mark.parametrize("gm,gn", [(2, 2), (3, 1), (1, 3)])
def test_grid_cuda_against_oracle(gm, gn):
    spec = stc.parse_benchmark_line(LINE)
    a, b, c0 = _host(spec, 31)
    A, B = a.to_device(), b.to_device()
    C = c0.to_device()
    ref = c0.copy()
    for rank in range(gm * gn):
        blk, _ = shard.contract_grid(spec, A, B, C, 2, "abc", rank, gm, gn)
        shard.contract_grid(spec, a, b, ref, 2, "abc", rank, gm, gn, contract_fn=_oracle_fn(2, "abc"))
        got = stc.DenseTensor(c0.extents, c0.strides, C.data.cpu().numpy())
        err = oracle.relative_error(shard.block_tensor(got, spec.labels_c, blk), shard.block_tensor(ref, spec.labels_c, blk))
        assert err <= TOL, (rank, err)
    got = stc.DenseTensor(c0.extents, c0.strides, C.data.cpu().numpy())
    assert oracle.relative_error(got, _classical(spec, a, b, c0)) <= TOL


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _nccl_worker(rank, world, port, ret):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    spec = stc.parse_benchmark_line(LINE)
    a, b, c0 = _host(spec)
    dev = torch.device("cuda", rank)
    A, B, C = a.to_device(dev), b.to_device(dev), c0.to_device(dev)
    shard.contract_sharded(spec, A, B, C, 2, "abc", rank, world)
    shard.gather_shards(spec, C, rank, world)
    ret[rank] = C.data.cpu().numpy()
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_nccl_nsplit_against_oracle():
    import torch
    import torch.multiprocessing as mp

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (the n-split over NCCL)")
    world = 2
    ret = mp.Manager().dict()
    mp.spawn(_nccl_worker, args=(world, _free_port(), ret), nprocs=world, join=True)
    spec = stc.parse_benchmark_line(LINE)
    a, b, c0 = _host(spec)
    ref = _classical(spec, a, b, c0)
    for r in range(world):
        got = stc.DenseTensor(c0.extents, c0.strides, ret[r])
        assert oracle.relative_error(got, ref) <= TOL, r


@pytest.mark.parametrize("gather", [True, False])
def test_contract_devices_one_process(gather):
    # stc_contract_sharded (one process driving several devices): here two "devices" that
    # are the same GPU with separate copies of A, B, C -- the shards share no data; the
    # gather is the device-to-device copy of each shard's block into the other copy of C.
    # Integer data: every path is exact, so each C copy equals the oracle's classical result
    # (gather) or holds exactly its own shard's block of it (no gather).
    import torch

    spec = stc.parse_benchmark_line("abij abef efij & a:8;b:16;i:12;j:16;e:8;f:16;")

    def ints(labels, seed):
        e = spec.tensor_extents(labels)
        return stc.DenseTensor(e, _rm(e), np.random.default_rng(seed).integers(-16, 17, int(np.prod(e))).astype(
            np.float64))

    a, b, c0 = ints(spec.labels_a, 61), ints(spec.labels_b, 62), ints(spec.labels_c, 63)
    ref = c0.copy()
    oracle.contract_reference(spec, a, b, ref)
    for level, variant in ((1, "abc"), (2, "abc"), (2, "ab")):
        A = [a.to_device(), a.to_device()]
        B = [b.to_device(), b.to_device()]
        C = [c0.to_device(), c0.to_device()]
        st = shard.contract_devices(spec, A, B, C, level, variant, [0, 0], gather=gather)
        assert st.pieces == 2 and st.leaf_multiplies == 7 ** level
        shards = shard.plan_shards(spec, c0, 2)
        for g in range(2):
            got = C[g].to_host()
            if gather:
                assert np.array_equal(got.data, ref.data), (level, variant, g)
            else:  # its own block contracted, the other block untouched
                for h, sh in enumerate(shards):
                    v = shard.shard_tensor(got, spec.labels_c, sh)
                    w = shard.shard_tensor(ref if h == g else c0, spec.labels_c, sh)
                    vv = np.lib.stride_tricks.as_strided(got.data[v.base_offset:], v.extents,
                                                         [s * 8 for s in v.strides])
                    ww = np.lib.stride_tricks.as_strided((ref if h == g else c0).data[w.base_offset:], w.extents,
                                                         [s * 8 for s in w.strides])
                    assert np.array_equal(vv, ww), (level, variant, g, h)
        del A, B, C
        torch.cuda.empty_cache()
