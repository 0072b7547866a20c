"""Counter-based synthetic inputs (numpy mirror) -- TEST INFRASTRUCTURE ONLY.

The BASELINE configs draw entries "uniform[-1,1] from seed".  For the big configs
(cfg3 at its literal extents: B is 32 GiB; cfg5: 8 GiB per operand, one copy per
rank) a sequential numpy generator would have to run over whole tensors on the
host of every rank.  A counter-based generator gives every element a value that
depends only on (seed, flat index of the element in the FULL tensor), so any
shard of a tensor can be generated on its own -- on the device by the library's
``stc_fill_uniform`` (csrc/stc_kernels.cu, used by bench.py and the GPU tests) or
here in numpy (used by tests/golden/make_big_golden.py to feed the reference, and
by the tests to check the device generator bitwise).

    key      = mix(seed + G)                                  (splitmix64, state = seed)
    u(j)     = mix(key + (j + 1) * G)                          (uint64 arithmetic mod 2^64)
    value(j) = (u(j) >> 11) * 2^-52 - 1.0                      in [-1, 1), 53-bit grid, exact

with G = 0x9E3779B97F4A7C15 and mix = the splitmix64 finaliser.  Every step is
exact in IEEE double, so numpy and CUDA produce identical bits.
"""

from __future__ import annotations

import numpy as np

__all__ = ["uniform_at", "tensor_values", "GOLDEN"]

GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK = (1 << 64) - 1


def _mix_int(z: int) -> int:
    z &= _MASK
    z = ((z ^ (z >> 30)) * _M1) & _MASK
    z = ((z ^ (z >> 27)) * _M2) & _MASK
    return z ^ (z >> 31)


def _mix(z: np.ndarray) -> np.ndarray:
    z ^= z >> np.uint64(30)
    z *= np.uint64(_M1)
    z ^= z >> np.uint64(27)
    z *= np.uint64(_M2)
    z ^= z >> np.uint64(31)
    return z


def uniform_at(seed: int, idx) -> np.ndarray:
    """value(j) for every flat index j in ``idx`` (any integer array)."""
    key = np.uint64(_mix_int(int(seed) + GOLDEN))
    with np.errstate(over="ignore"):
        z = np.asarray(idx).astype(np.uint64, copy=True)
        z += np.uint64(1)
        z *= np.uint64(GOLDEN)
        z += key
        z = _mix(z)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -52) - 1.0


def tensor_values(seed: int, extents, strides=None, base: int = 0, chunk: int = 1 << 24) -> np.ndarray:
    """Compact row-major array over ``extents`` whose element at multi-index
    (i_0, ..., i_{d-1}) is value(base + sum i_d * strides[d]).  ``strides`` default
    to the row-major strides of ``extents`` (a whole tensor); pass the full
    tensor's strides and a base offset to generate a slice of it."""
    ext = tuple(int(e) for e in extents)
    if strides is None:
        strides, run = [], 1
        for e in reversed(ext):
            strides.append(run)
            run *= e
        strides = tuple(reversed(strides))
    n = int(np.prod(ext)) if ext else 1
    out = np.empty(n, dtype=np.float64)
    if n == 0:
        return out
    # row-major decomposition of the compact position, chunk by chunk
    inner = [1] * len(ext)
    for d in range(len(ext) - 2, -1, -1):
        inner[d] = inner[d + 1] * ext[d + 1]
    for s in range(0, n, chunk):
        pos = np.arange(s, min(n, s + chunk), dtype=np.int64)
        flat = np.full(pos.shape, int(base), dtype=np.int64)
        for d in range(len(ext)):
            flat += ((pos // inner[d]) % ext[d]) * int(strides[d])
        out[s:s + pos.size] = uniform_at(seed, flat)
    return out
