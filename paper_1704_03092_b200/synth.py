"""Seeded synthetic operands generated in HBM (bench.py and the GPU tests).

The BASELINE configs fix only "entries uniform[-1,1] from seed".  For the large
ones (cfg5: three 8 GiB operands; cfg3 at its literal extents: a 32 GiB B) the
inputs are produced on the device by ``stc_fill_uniform`` (C ABI), a
counter-based generator whose value for an element depends only on the seed and
the element's flat index in the full tensor: a rank can generate exactly its
shard of B and C, and the host-side mirror in ``oracle/synth.py`` (used to feed
the reference when the golden fixtures are made) gives the same bits.
"""

from __future__ import annotations

import ctypes

from . import _lib
from .tensor import DenseTensor

__all__ = ["fill_uniform", "uniform_tensor", "row_major"]


def row_major(extents) -> tuple:
    out, run = [], 1
    for e in reversed(tuple(extents)):
        out.append(run)
        run *= int(e)
    return tuple(reversed(out))


def fill_uniform(out, seed: int, extents, strides=None, base: int = 0, stream=None) -> None:
    """Fill the compact CUDA float64 tensor ``out`` (row-major over ``extents``)
    with value(seed, base + sum i_d * strides[d]); ``strides`` default to the
    row-major strides of ``extents`` (a whole tensor)."""
    import torch

    ext = tuple(int(e) for e in extents)
    st = row_major(ext) if strides is None else tuple(int(s) for s in strides)
    if not (torch.is_tensor(out) and out.is_cuda and out.dtype == torch.float64 and out.is_contiguous()):
        raise ValueError("out must be a contiguous float64 CUDA tensor")
    n = 1
    for e in ext:
        n *= e
    if out.numel() < n:
        raise ValueError(f"out holds {out.numel()} elements, the shape needs {n}")
    E = (ctypes.c_int64 * max(len(ext), 1))(*ext)
    S = (ctypes.c_int64 * max(len(st), 1))(*st)
    s = stream if stream is not None else torch.cuda.current_stream(out.device)
    with torch.cuda.device(out.device):
        _lib.check(_lib.lib().stc_fill_uniform(ctypes.c_void_p(out.data_ptr()), len(ext), E, S, int(base),
                                               ctypes.c_uint64(int(seed) & ((1 << 64) - 1)),
                                               ctypes.c_void_p(s.cuda_stream)))


def uniform_tensor(seed: int, extents, device, full_strides=None, base: int = 0) -> DenseTensor:
    """A compact row-major DenseTensor in HBM over ``extents`` holding the
    generator's values; with ``full_strides``/``base`` it is that slice of a
    larger tensor (e.g. a rank's n-shard of B or C)."""
    import torch

    ext = tuple(int(e) for e in extents)
    n = 1
    for e in ext:
        n *= e
    data = torch.empty(max(n, 1), dtype=torch.float64, device=device)
    fill_uniform(data, seed, ext, full_strides, base)
    return DenseTensor(ext, row_major(ext), data)
