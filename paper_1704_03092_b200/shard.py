"""Multi-GPU splits (north-star subsystem 5).

n-split: the J bundle (columns of B and C) of a contraction is split into
contiguous ranges of one of its labels; every rank contracts its range
independently -- A is shared, B and C are sliced -- so there is no reduction.
2-D split (plan_grid / contract_grid): an I label and a J label are split on a
gm x gn rank grid, so a rank holds A[I_r, :], B[:, J_c] and C[I_r, J_c] -- the
operand replication of the n-split (all of A on every rank) drops to 1/gm of A
and 1/gn of B; still no reduction, since every C element is owned by one rank.
One process per GPU, torch.distributed for the plumbing; the only collective
is the optional all-gather of the C blocks (NCCL over NVLink on GPUs, gloo on
CPUs).  The reference has no distributed path; the
paper's MPI/CTF runs are the analogue.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .tensor import ContractionSpec, DenseTensor

__all__ = ["Shard", "plan_shards", "shard_tensor", "shard_spec", "contract_sharded", "gather_shards", "Block",
           "plan_grid", "block_spec", "block_tensor", "contract_grid", "gather_blocks", "contract_devices"]


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


def _storage(c: DenseTensor):
    import torch

    return c.data if isinstance(c.data, torch.Tensor) else torch.from_numpy(c.data)


def _region(c: DenseTensor, labels: str, sh: Shard):
    """Strided torch view of the shard region of C (label order of C)."""
    import torch

    v = shard_tensor(c, labels, sh)
    return torch.as_strided(_storage(c), v.extents, v.strides, v.base_offset)


def gather_shards(spec: ContractionSpec, c: DenseTensor, rank: int, world: int, label: str | None = None,
                  group=None) -> None:
    """All-gather every rank's C shard into this rank's full C (in place).

    One collective: every rank contributes its shard as one dense block, padded
    to the largest shard (all_gather needs equal sizes; plan_shards' ranges may
    differ by one), into a shard-major [world, size] buffer
    (all_gather_into_tensor: NCCL over NVLink for CUDA storage, gloo for host
    storage); each received block is then written into its strided region of C
    with one copy.  Extra memory: the buffer, one C's worth.
    """
    import torch
    import torch.distributed as dist

    shards = plan_shards(spec, c, world, label)
    regions = [_region(c, spec.labels_c, s) for s in shards]
    size = max(r.numel() for r in regions)
    data = _storage(c)
    # gloo moves host tensors: device storage is staged through host memory
    staging = "cpu" if dist.get_backend(group) == "gloo" else data.device
    flat = torch.zeros(size, dtype=data.dtype, device=staging)
    flat[: regions[rank].numel()].view(regions[rank].shape).copy_(regions[rank])
    out = torch.empty(world * size, dtype=data.dtype, device=staging)
    if dist.get_backend(group) != "gloo":
        dist.all_gather_into_tensor(out, flat, group=group)
    else:  # gloo has no all_gather_into_tensor: the list form over views of the same buffer
        dist.all_gather(list(out.view(world, size).unbind(0)), flat, group=group)
    for s, (sh, reg) in enumerate(zip(shards, regions)):
        if s != rank:
            reg.copy_(out[s * size: s * size + reg.numel()].view(reg.shape))


# ---------------------------------------------------------------- 2-D split
@dataclass(frozen=True)
class Block:
    """One rank's block of a gm x gn grid: a range of an I label and of a J label."""
    row: Shard   # I-bundle label range (rows of A and C)
    col: Shard   # J-bundle label range (columns of B and C)


def _pick(spec: ContractionSpec, t: DenseTensor, labels: str, bundle: str, parts: int, what: str) -> str:
    cand = [l for l in bundle if spec.extents[l] >= parts]
    if not cand:
        raise ValueError(f"no {what} label has extent >= {parts}")
    stride = lambda l: abs(t.strides[labels.index(l)])
    return max(cand, key=lambda l: (spec.extents[l] % parts == 0, stride(l)))


def _ranges(label: str, ext: int, parts: int) -> list:
    base, extra = divmod(ext, parts)
    out, s = [], 0
    for r in range(parts):
        n = base + (1 if r < extra else 0)
        out.append(Shard(label, s, s + n))
        s += n
    return out


def plan_grid(spec: ContractionSpec, c: DenseTensor, gm: int, gn: int, row_label: str | None = None,
              col_label: str | None = None) -> list:
    """Blocks of a gm x gn grid, rank r -> (r // gn, r % gn): an I label cut into gm
    contiguous ranges and a J label into gn (sizes within 1).  Default labels: the
    largest C stride among the bundle's labels with extent >= the part count,
    preferring divisible extents (as plan_shards)."""
    if gm < 1 or gn < 1:
        raise ValueError("grid dimensions must be positive")
    if gm > 1 and not spec.bundle_i:
        raise ValueError("the I bundle is empty: nothing to split")
    if gn > 1 and not spec.bundle_j:
        raise ValueError("the J bundle is empty: nothing to split")
    if gm > 1 or row_label is not None:
        row_label = row_label or _pick(spec, c, spec.labels_c, spec.bundle_i, gm, "I")
        if row_label not in spec.bundle_i:
            raise ValueError(f"label {row_label!r} is not in the I bundle {spec.bundle_i!r}")
    if gn > 1 or col_label is not None:
        col_label = col_label or _pick(spec, c, spec.labels_c, spec.bundle_j, gn, "J")
        if col_label not in spec.bundle_j:
            raise ValueError(f"label {col_label!r} is not in the J bundle {spec.bundle_j!r}")
    rows = _ranges(row_label, spec.extents[row_label], gm) if row_label else [Shard("", 0, 0)] * gm
    cols = _ranges(col_label, spec.extents[col_label], gn) if col_label else [Shard("", 0, 0)] * gn
    return [Block(rows[r // gn], cols[r % gn]) for r in range(gm * gn)]


def block_spec(spec: ContractionSpec, blk: Block) -> ContractionSpec:
    ext = dict(spec.extents)
    for sh in (blk.row, blk.col):
        if sh.label:
            ext[sh.label] = sh.stop - sh.start
    return ContractionSpec(spec.labels_c, spec.labels_a, spec.labels_b, ext)


def block_tensor(t: DenseTensor, labels: str, blk: Block) -> DenseTensor:
    """View of `t` restricted to the block's label ranges it carries (same storage)."""
    for sh in (blk.row, blk.col):
        if sh.label:
            t = shard_tensor(t, labels, sh)
    return t


def contract_grid(spec: ContractionSpec, a: DenseTensor, b: DenseTensor, c: DenseTensor, level: int, variant,
                  rank: int, gm: int, gn: int, row_label: str | None = None, col_label: str | None = None,
                  contract_fn=None, **kw):
    """Contract this rank's block of C (in place): A rows, B columns and C block of
    the rank's grid cell.  `contract_fn` as in contract_sharded; returns (block, stats)."""
    if contract_fn is None:
        from .strassen import contract as contract_fn
    blk = plan_grid(spec, c, gm, gn, row_label, col_label)[rank]
    st = contract_fn(block_spec(spec, blk), block_tensor(a, spec.labels_a, blk), block_tensor(b, spec.labels_b, blk),
                     block_tensor(c, spec.labels_c, blk), level, variant, **kw)
    return blk, st


def gather_blocks(spec: ContractionSpec, c: DenseTensor, rank: int, gm: int, gn: int, row_label: str | None = None,
                  col_label: str | None = None, group=None) -> None:
    """All-gather every rank's C block into this rank's full C (in place)."""
    import torch
    import torch.distributed as dist

    blocks = plan_grid(spec, c, gm, gn, row_label, col_label)
    data = c.data if isinstance(c.data, torch.Tensor) else torch.from_numpy(c.data)

    def dense(blk):
        v = block_tensor(c, spec.labels_c, blk)
        return torch.as_strided(data, v.extents, v.strides, v.base_offset)

    mine = dense(blocks[rank]).contiguous()
    # all_gather needs equal sizes: pad every block to the largest one
    size = max(int(np.prod(block_tensor(c, spec.labels_c, b).extents)) for b in blocks)
    flat = torch.zeros(size, dtype=mine.dtype, device=mine.device)
    flat[: mine.numel()] = mine.reshape(-1)
    bufs = [torch.empty_like(flat) for _ in blocks]
    dist.all_gather(bufs, flat, group=group)
    for blk, buf in zip(blocks, bufs):
        d = dense(blk)
        d.copy_(buf[: d.numel()].reshape(d.shape))


# ---------------------------------------------------------------- one process, several GPUs
def contract_devices(spec: ContractionSpec, a: list, b: list, c: list, level: int, variant, devices: list,
                     label: str | None = None, gather: bool = True):
    """The n-split driven from one process (C ABI stc_contract_sharded).

    a[g], b[g], c[g]: device g's copies (DenseTensors with CUDA storage on
    devices[g], the full tensors' layouts); shard g of C (plan_shards order) is
    contracted on devices[g], and with `gather` every device's C then gets the
    other shards' blocks by peer copies over NVLink -- no collective library.
    Synchronises the devices' current streams before returning; returns the
    summed RunStats (pieces = number of devices).
    """
    import ctypes

    import torch

    from . import _lib
    from .stats import RunStats
    from .strassen import _variant, problem_of

    n = len(devices)
    if not (len(a) == len(b) == len(c) == n) or n < 1:
        raise ValueError("one A, B and C per device")
    for t in (*a, *b, *c):
        if not (isinstance(t.data, torch.Tensor) and t.data.is_cuda):
            raise ValueError("contract_devices takes device (CUDA) storage")
    lab = -1 if label is None else spec.bundle_j.index(label)
    prob = problem_of(spec, a[0], b[0], c[0], level, _variant(variant))
    L = _lib.lib()
    need = ctypes.c_size_t()
    _lib.check(L.stc_sharded_workspace_size(ctypes.byref(prob), n, lab, ctypes.byref(need)))
    ws = [torch.empty(max(int(need.value), 256), dtype=torch.uint8, device=t.data.device) for t in c]
    streams = [torch.cuda.current_stream(t.data.device) for t in c]

    def ptrs(xs):
        return (ctypes.c_void_p * n)(*[x.data_ptr() for x in xs])

    st = _lib.Stats()
    _lib.check(L.stc_contract_sharded(ctypes.byref(prob), n, (ctypes.c_int * n)(*devices), lab,
                                      ptrs([t.data for t in a]), ptrs([t.data for t in b]),
                                      ptrs([t.data for t in c]), ptrs(ws),
                                      (ctypes.c_size_t * n)(*[w.numel() for w in ws]),
                                      (ctypes.c_void_p * n)(*[s.cuda_stream for s in streams]), int(gather),
                                      ctypes.byref(st)))
    for s in streams:
        s.synchronize()
    out = RunStats()
    out.absorb(st)
    return out
