"""Multi-GPU n-bundle split (north-star subsystem 5).

The J bundle (columns of B and C) of a contraction is split into contiguous
ranges of one of its labels; every rank contracts its range independently --
A is shared, B and C are sliced -- so there is no reduction.  One process per
GPU, torch.distributed for the plumbing; the only collective is the optional
all-gather of the C shards (NCCL over NVLink on GPUs, gloo on CPUs).  The
reference has no distributed path; the paper's MPI/CTF runs are the
analogue.
"""

from __future__ import annotations

from dataclasses import dataclass

from .tensor import ContractionSpec, DenseTensor

__all__ = ["Shard", "plan_shards", "shard_tensor", "shard_spec", "contract_sharded", "gather_shards"]


@dataclass(frozen=True)
class Shard:
    label: str   # J-bundle label that is split
    start: int   # [start, stop) of that label owned by the rank
    stop: int


def plan_shards(spec: ContractionSpec, c: DenseTensor, world: int, label: str | None = None) -> list:
    """Split one J label into `world` contiguous ranges (sizes differ by at most 1).

    Default label: the J label with the largest stride in C whose extent is at
    least `world` (each shard is then one contiguous slab of C), preferring
    extents divisible by `world`.
    """
    if world < 1:
        raise ValueError("world size must be positive")
    if not spec.bundle_j:
        raise ValueError("the J bundle is empty: nothing to split")
    if label is None:
        cand = [l for l in spec.bundle_j if spec.extents[l] >= world]
        if not cand:
            raise ValueError(f"no J label has extent >= {world}")
        stride = lambda l: abs(c.strides[spec.labels_c.index(l)])
        label = max(cand, key=lambda l: (spec.extents[l] % world == 0, stride(l)))
    if label not in spec.bundle_j:
        raise ValueError(f"label {label!r} is not in the J bundle {spec.bundle_j!r}")
    ext = spec.extents[label]
    base, extra = divmod(ext, world)
    out, s = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append(Shard(label, s, s + n))
        s += n
    return out


def shard_spec(spec: ContractionSpec, sh: Shard) -> ContractionSpec:
    ext = dict(spec.extents)
    ext[sh.label] = sh.stop - sh.start
    return ContractionSpec(spec.labels_c, spec.labels_a, spec.labels_b, ext)


def shard_tensor(t: DenseTensor, labels: str, sh: Shard) -> DenseTensor:
    """View of `t` restricted to the shard's range of its label (same storage)."""
    if sh.label not in labels:
        return t
    ax = labels.index(sh.label)
    ext = list(t.extents)
    ext[ax] = sh.stop - sh.start
    return DenseTensor(tuple(ext), t.strides, t.data, t.base_offset + sh.start * t.strides[ax])


def contract_sharded(spec: ContractionSpec, a: DenseTensor, b: DenseTensor, c: DenseTensor, level: int, variant,
                     rank: int, world: int, label: str | None = None, contract_fn=None, **kw):
    """Contract this rank's shard of C (in place, on this rank's storage).

    `contract_fn(spec, a, b, c, level, variant, **kw)` defaults to the B200
    `contract`; returns (shard, stats).
    """
    if contract_fn is None:
        from .strassen import contract as contract_fn
    sh = plan_shards(spec, c, world, label)[rank]
    sp = shard_spec(spec, sh)
    st = contract_fn(sp, a, shard_tensor(b, spec.labels_b, sh), shard_tensor(c, spec.labels_c, sh), level, variant,
                     **kw)
    return sh, st


def _pack(c: DenseTensor, labels: str, sh: Shard):
    """Dense copy of the shard region of C (label order of C, first axis slowest)."""
    import torch

    v = shard_tensor(c, labels, sh)
    data = c.data if isinstance(c.data, torch.Tensor) else torch.from_numpy(c.data)
    return torch.as_strided(data, v.extents, v.strides, v.base_offset).contiguous()


def gather_shards(spec: ContractionSpec, c: DenseTensor, rank: int, world: int, label: str | None = None,
                  group=None) -> None:
    """All-gather every rank's C shard into this rank's full C (in place).

    Shards are exchanged as dense blocks with torch.distributed.all_gather (NCCL
    for CUDA storage, gloo for host storage) and scattered back into C's layout.
    """
    import torch
    import torch.distributed as dist

    shards = plan_shards(spec, c, world, label)
    mine = _pack(c, spec.labels_c, shards[rank])
    blocks = [torch.empty_like(_pack(c, spec.labels_c, s)) for s in shards]
    dist.all_gather(blocks, mine, group=group)
    data = c.data if isinstance(c.data, torch.Tensor) else torch.from_numpy(c.data)
    for s, blk in zip(shards, blocks):
        v = shard_tensor(c, spec.labels_c, s)
        torch.as_strided(data, v.extents, v.strides, v.base_offset).copy_(blk)
