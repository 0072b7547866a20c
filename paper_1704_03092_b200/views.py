"""Device-resident block-scatter views and the kernel-level API.

Reference counterparts (``/root/reference/pkg/src/strassen_tc``):

* ``BlockScatterView``, ``make_view``, ``matrix_view``, ``split_view``,
  ``pad_view`` -- scatter.py:43-165.  Here the scatter vectors (``rscat``,
  ``cscat``) and block-scatter vectors (``rbs``, ``cbs``) are int64 CUDA
  tensors built by device kernels (``stc_bundle_scatter``,
  ``stc_block_vector``): north-star subsystem (1).
* ``quadrant_views`` -- strassen.py:101-127.
* ``OperandTermSide`` / ``FusedPrimitive`` / ``run_fused`` /
  ``run_gemm_dense`` -- kernels.py:102-154, driver.py:26-152: one fused
  Strassen term on the DMMA kernel (subsystems (2)+(3)).
* ``PackedBuffer`` / ``pack_a`` / ``pack_b`` / ``microkernel`` -- kernels.py:67-233: the
  packing pass and the micro-tile as standalone device calls (``stc_pack_panel``,
  ``stc_microtile``), bitwise the reference's panels and tiles.  ``contract`` does this
  work inside the fused kernel; these exist for callers of the component API.
* ``accumulate_dense_to_view`` / ``unpack_to_dense`` -- kernels.py:236-264
  (subsystem (4)).
* ``relative_error`` -- oracle.py:110-124, reduced on the device.

Everything here runs on the GPU through the C ABI; nothing falls back to the
CPU.  ``BlockingParams`` is accepted for signature compatibility (the GPU
tile configuration is fixed, see ``TILE``).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .stats import RunStats
from .tensor import DenseTensor

__all__ = [
    "PAD",
    "TILE",
    "BlockingParams",
    "CTA_TILES",
    "TileConfig",
    "DEFAULT_BLOCKING",
    "BlockScatterView",
    "FusedPrimitive",
    "OperandTermSide",
    "PackedBuffer",
    "accumulate_dense_to_view",
    "make_view",
    "matrix_view",
    "microkernel",
    "pack_a",
    "pack_b",
    "pad_view",
    "quadrant_views",
    "relative_error",
    "run_fused",
    "run_gemm_dense",
    "split_view",
    "unpack_to_dense",
]

PAD = _lib.PAD

# GPU tiling of the fused DMMA kernel (csrc/stc_fused.cu), the counterpart of the
# reference's BlockingParams: chosen per problem by the planner; TileConfig (below)
# requests a CTA tile shape and caps the ring depth per call.
TILE = {
    "cta_tile": (128, 128),              # 64 x 256 / 256 x 64 for 64-wide quadrants, 64 x 128 for small problems
    "warp_tile": (64, 32),               # 8 consumer warps (32 x 32 on the 64 x 128 tiles), m16n8k4.f64 (DMMA)
    "k_chunk": 8,                        # one TMA box per view per stage: 128 x 8 doubles
    "stages": "8 with one view per side (L0, pre-summed or Naive slots); 6 / 3 with 2 / 4 views per side",
    "producer_warps": 4,                 # warp 0 issues the TMA loads, warps 1-3 run the C epilogue
    "summing_warps": 4,                  # in-kernel operand sums (L >= 1 without pre-summed slots)
    "mma": "mma.sync.m16n8k4.row.col.f64 (SASS DMMA.8x8x4)",
    "gather_kernel": {"cta_tile": (128, 128), "k_chunk": 16, "stages": 3},  # k_strassen_gemm (force_slow, reference tiling, L >= 4)
}


@dataclass(frozen=True)
class BlockingParams:
    """The reference's cache/register blocking (kernels.py:34-56).

    Validated exactly like the reference and used as the block geometry of
    views (rb/cb); the B200 kernel's own tiling is ``TILE``.
    """

    mc: int = 96
    nc: int = 4096
    kc: int = 256
    mr: int = 8
    nr: int = 4
    kr: int = 4

    def __post_init__(self):
        for name in ("mc", "nc", "kc", "mr", "nr", "kr"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be positive")
        if self.mc % self.mr or self.nc % self.nr or self.kc % self.kr:
            raise ValueError(
                f"cache blocks must be multiples of register blocks: mc={self.mc} mr={self.mr} "
                f"nc={self.nc} nr={self.nr} kc={self.kc} kr={self.kr}")


DEFAULT_BLOCKING = BlockingParams()

# CTA tile shapes of the fused kernel, (rows of I, columns of J) -> stc_fused.cu Shape<ts>
CTA_TILES = {(128, 128): 0, (64, 256): 1, (256, 64): 2, (64, 128): 3, (128, 64): 4}


@dataclass(frozen=True)
class TileConfig:
    """The GPU tile config that replaces the reference's ``BlockingParams``
    (kernels.py:34-56) as ``contract(..., params=...)``.

    ``cta_tile``: the fused DMMA kernel's CTA tile (a key of ``CTA_TILES``), None
    for the planner's choice; ``stages``: a cap on its TMA ring depth (2..8), None
    for the most that fit in shared memory.  Like the reference's blocking it
    only changes how the work is scheduled: every tile and depth gives bitwise the
    same C (the DMMA k-steps of an element run in the same order).  A shape the
    problem cannot use raises ValueError before any device work (the shaped tiles
    need L >= 1 and a non-Naive variant).  ``BlockingParams`` (the reference's
    CPU blocking) is still accepted and leaves every choice to the planner.
    """

    cta_tile: tuple | None = None
    stages: int | None = None

    def __post_init__(self):
        if self.cta_tile is not None:
            object.__setattr__(self, "cta_tile", tuple(int(v) for v in self.cta_tile))
            if self.cta_tile not in CTA_TILES:
                raise ValueError(f"cta_tile must be one of {sorted(CTA_TILES)}, got {self.cta_tile}")
        if self.stages is not None and not 2 <= int(self.stages) <= 8:
            raise ValueError(f"stages must be in 2..8, got {self.stages}")

    @property
    def code(self) -> int:
        """stc_problem.tiling: STC_TILING(1 + shape, stages) (include/stc_b200.h)."""
        shape = 0 if self.cta_tile is None else 1 + CTA_TILES[self.cta_tile]
        return shape | ((self.stages or 0) << 4)


def tiling_code(params) -> int:
    """stc_problem.tiling for contract()'s ``params``: a TileConfig's request, 0
    (the planner) for the reference's BlockingParams."""
    if isinstance(params, TileConfig):
        return params.code
    if not all(hasattr(params, f) for f in ("mc", "nc", "kc", "mr", "nr", "kr")):
        raise TypeError("params must be a TileConfig (GPU tiling) or a BlockingParams (the reference's blocking)")
    return 0


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 contraction path has no CPU fallback")
    return torch


def _stream():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _device_of(t: DenseTensor):
    if not t.on_device:
        raise ValueError("device views need HBM-resident storage (use DenseTensor.to_device())")
    return t.data.device


def _scatter(extents, strides, base, device):
    """Device-built scatter vector of one bundle (scatter.py:105-112)."""
    torch = _torch()
    n = int(np.prod(extents, dtype=np.int64)) if len(extents) else 1
    out = torch.empty(n, dtype=torch.int64, device=device)
    b = _lib.Bundle.of(extents, strides)
    with torch.cuda.device(device):
        _lib.check(_lib.lib().stc_bundle_scatter(ctypes.byref(b), int(base), n, _ptr(out), _stream()))
    return out


def _block_vector(scat, blk: int, unit: int):
    """Device-built block-scatter vector (scatter.py:26-40)."""
    torch = _torch()
    scat = scat.contiguous()
    nb = -(-scat.numel() // blk)
    out = torch.empty(nb, dtype=torch.int64, device=scat.device)
    with torch.cuda.device(scat.device):
        _lib.check(_lib.lib().stc_block_vector(_ptr(scat), scat.numel(), int(blk), int(unit), _ptr(out), _stream()))
    return out


@dataclass(eq=False)
class BlockScatterView:
    """m x n matrix view of ``base``: element (i, j) at data[rscat[i] + cscat[j]]."""

    base: DenseTensor
    m: int
    n: int
    rscat: object
    cscat: object
    rb: int
    cb: int
    rbs: object
    cbs: object
    row_unit_stride: int = 1
    col_unit_stride: int = 1

    @classmethod
    def from_scatter(cls, base, rscat, cscat, rb, cb, row_unit_stride=1, col_unit_stride=1):
        torch = _torch()
        if rb < 1 or cb < 1:
            raise ValueError("block sizes must be >= 1")
        dev = _device_of(base)
        rscat = torch.as_tensor(rscat, dtype=torch.int64, device=dev).contiguous()
        cscat = torch.as_tensor(cscat, dtype=torch.int64, device=dev).contiguous()
        return cls(base=base, m=rscat.numel(), n=cscat.numel(), rscat=rscat, cscat=cscat, rb=rb, cb=cb,
                   rbs=_block_vector(rscat, rb, row_unit_stride), cbs=_block_vector(cscat, cb, col_unit_stride),
                   row_unit_stride=row_unit_stride, col_unit_stride=col_unit_stride)

    def get(self, i: int, j: int) -> float:
        r, c = int(self.rscat[i]), int(self.cscat[j])
        if r == PAD or c == PAD:
            return 0.0
        return float(self.base.data[r + c])

    def set(self, i: int, j: int, value: float) -> None:
        r, c = int(self.rscat[i]), int(self.cscat[j])
        if r == PAD or c == PAD:
            return
        self.base.data[r + c] = value

    def to_dense(self):
        """Materialise the view (PAD reads 0) as a column-major device matrix."""
        return unpack_to_dense(OperandTermSide([self], [1]))

    def __eq__(self, other) -> bool:
        torch = _torch()
        return (isinstance(other, BlockScatterView) and self.base is other.base
                and (self.m, self.n, self.rb, self.cb) == (other.m, other.n, other.rb, other.cb)
                and torch.equal(self.rscat, other.rscat) and torch.equal(self.cscat, other.cscat)
                and torch.equal(self.rbs, other.rbs) and torch.equal(self.cbs, other.cbs))


def make_view(t: DenseTensor, row_bundle, col_bundle, label_axes, rb: int, cb: int) -> BlockScatterView:
    """Matricise ``t`` (scatter.py:115-131); base_offset folded into cscat."""
    row_axes = [label_axes[l] for l in row_bundle]
    col_axes = [label_axes[l] for l in col_bundle]
    if set(row_axes) & set(col_axes):
        raise ValueError("row and column bundles overlap")
    if sorted(row_axes + col_axes) != list(range(t.ndim)):
        raise ValueError("bundles must cover every axis of the tensor exactly once")
    dev = _device_of(t)
    rscat = _scatter([t.extents[a] for a in row_axes], [t.strides[a] for a in row_axes], 0, dev)
    cscat = _scatter([t.extents[a] for a in col_axes], [t.strides[a] for a in col_axes], t.base_offset, dev)
    row_unit = t.strides[row_axes[0]] if row_axes else 1
    col_unit = t.strides[col_axes[0]] if col_axes else 1
    return BlockScatterView.from_scatter(t, rscat, cscat, rb, cb, row_unit, col_unit)


def matrix_view(t: DenseTensor, rb: int, cb: int) -> BlockScatterView:
    """A 2-axis tensor viewed as itself (scatter.py:134-140)."""
    if t.ndim != 2:
        raise ValueError(f"matrix_view needs a 2-axis tensor, got {t.ndim}")
    dev = _device_of(t)
    rscat = _scatter([t.extents[0]], [t.strides[0]], 0, dev)
    cscat = _scatter([t.extents[1]], [t.strides[1]], t.base_offset, dev)
    return BlockScatterView.from_scatter(t, rscat, cscat, rb, cb, t.strides[0], t.strides[1])


def split_view(v: BlockScatterView, row_range, col_range) -> BlockScatterView:
    """Sub-view over half-open ranges, blocks re-aligned (scatter.py:143-152)."""
    r0, r1 = row_range
    c0, c1 = col_range
    if not (0 <= r0 < r1 <= v.m and 0 <= c0 < c1 <= v.n):
        raise ValueError(f"empty or out-of-bounds range ({row_range}, {col_range}) for {v.m}x{v.n} view")
    return BlockScatterView.from_scatter(v.base, v.rscat[r0:r1], v.cscat[c0:c1], v.rb, v.cb,
                                         v.row_unit_stride, v.col_unit_stride)


def pad_view(v: BlockScatterView, m_target: int, n_target: int) -> BlockScatterView:
    """Extend with PAD rows/columns (scatter.py:155-165)."""
    torch = _torch()
    if m_target < v.m or n_target < v.n:
        raise ValueError("pad targets must not shrink the view")
    if m_target == v.m and n_target == v.n:
        return v
    dev = v.rscat.device
    rscat = torch.cat([v.rscat, torch.full((m_target - v.m,), PAD, dtype=torch.int64, device=dev)])
    cscat = torch.cat([v.cscat, torch.full((n_target - v.n,), PAD, dtype=torch.int64, device=dev)])
    return BlockScatterView.from_scatter(v.base, rscat, cscat, v.rb, v.cb, v.row_unit_stride, v.col_unit_stride)


def quadrant_views(v: BlockScatterView, level: int) -> dict:
    """4^level congruent quadrants, ids row-major per level (strassen.py:101-127)."""
    if level < 1:
        raise ValueError(f"level must be >= 1, got {level}")
    step = 1 << level
    v = pad_view(v, -(-v.m // step) * step, -(-v.n // step) * step)

    def rec(view, lev):
        if lev == 0:
            return [view]
        h, w = view.m // 2, view.n // 2
        out = []
        for rr, cc in (((0, h), (0, w)), ((0, h), (w, 2 * w)), ((h, 2 * h), (0, w)), ((h, 2 * h), (w, 2 * w))):
            out.extend(rec(split_view(view, rr, cc), lev - 1))
        return out

    return dict(enumerate(rec(v, level)))


@dataclass(eq=False)
class OperandTermSide:
    """1..16 views over one parent with +/-1 coefficients (kernels.py:102-154)."""

    views: tuple
    coeffs: tuple
    _checked: bool = field(default=False, repr=False)

    def __post_init__(self):
        self.views = tuple(self.views)
        self.coeffs = tuple(int(c) for c in self.coeffs)
        if not self.views or len(self.views) != len(self.coeffs):
            raise ValueError("need equally many views and coefficients, at least one each")
        if any(c not in (-1, 1) for c in self.coeffs):
            raise ValueError(f"coefficients must be +/-1, got {self.coeffs}")
        v0 = self.views[0]
        for v in self.views:
            if (v.m, v.n, v.rb, v.cb) != (v0.m, v0.n, v0.rb, v0.cb):
                raise ValueError("views of one side must share matrix and block geometry")
            if v.base.data is not v0.base.data:
                raise ValueError("views of one side must share one parent tensor")
        if len(self.views) > 16:
            raise ValueError("at most 16 views per side on the device")

    @property
    def m(self) -> int:
        return self.views[0].m

    @property
    def n(self) -> int:
        return self.views[0].n

    @property
    def rb(self) -> int:
        return self.views[0].rb

    @property
    def cb(self) -> int:
        return self.views[0].cb

    @property
    def data(self):
        return self.views[0].base.data


@dataclass(eq=False)
class FusedPrimitive:
    """c_side targets += (sum a_side) (sum b_side) (driver.py:26-44)."""

    a_side: OperandTermSide
    b_side: OperandTermSide
    c_side: OperandTermSide

    def __post_init__(self):
        m, k = self.a_side.m, self.a_side.n
        n = self.b_side.n
        if self.b_side.m != k:
            raise ValueError(f"A is {m}x{k} but B is {self.b_side.m}x{n}")
        if (self.c_side.m, self.c_side.n) != (m, n):
            raise ValueError(f"C is {self.c_side.m}x{self.c_side.n}, expected {m}x{n}")

    @property
    def shape(self) -> tuple:
        return self.a_side.m, self.b_side.n, self.a_side.n


def _offsets_host(view: BlockScatterView) -> np.ndarray:
    r = view.rscat.cpu().numpy()
    c = view.cscat.cpu().numpy()
    r, c = r[r != PAD], c[c != PAD]
    return np.unique((r[:, None] + c[None, :]).ravel())


def check_c_targets(views) -> None:
    """Targets must be pairwise disjoint or identical (driver.py:53-61)."""
    offs = [_offsets_host(v) for v in views]
    for i in range(len(offs)):
        for j in range(i + 1, len(offs)):
            if offs[i].shape == offs[j].shape and np.array_equal(offs[i], offs[j]):
                continue
            if np.intersect1d(offs[i], offs[j], assume_unique=True).size:
                raise ValueError(f"C targets {i} and {j} overlap without being identical")


def _ptr_array(ts):
    arr = (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])
    return ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p)), arr


def _coeff_array(cs):
    arr = (ctypes.c_double * len(cs))(*[float(c) for c in cs])
    return arr


def run_fused(prim: FusedPrimitive, params: BlockingParams = DEFAULT_BLOCKING, stats: RunStats | None = None,
              threads: int = 1, force_slow: bool = False, workspace=None, validate: bool = False) -> RunStats:
    """One fused Strassen term on the DMMA kernel; counts one leaf multiply."""
    torch = _torch()
    if stats is None:
        stats = RunStats()
    if validate:
        check_c_targets(prim.c_side.views)
    m, n, k = prim.shape
    a, b, c = prim.a_side, prim.b_side, prim.c_side
    L = _lib.lib()
    need = ctypes.c_size_t()
    _lib.check(L.stc_fused_term_workspace_size(m, n, k, len(a.views), len(b.views), len(c.views), ctypes.byref(need)))
    ws = torch.empty(max(int(need.value), 1), dtype=torch.uint8, device=a.data.device)
    keep = []

    def side(s, rows_of, cols_of):
        pr, ar = _ptr_array([rows_of(v) for v in s.views])
        pc, ac = _ptr_array([cols_of(v) for v in s.views])
        co = _coeff_array(s.coeffs)
        keep.extend([ar, ac, co])
        return pr, pc, co

    a_r, a_c, a_co = side(a, lambda v: v.rscat, lambda v: v.cscat)
    b_r, b_c, b_co = side(b, lambda v: v.rscat, lambda v: v.cscat)
    c_r, c_c, c_co = side(c, lambda v: v.rscat, lambda v: v.cscat)
    st = _lib.Stats()
    flags = _lib.FLAG_FORCE_SLOW if force_slow else 0
    with torch.cuda.device(a.data.device):
        _lib.check(L.stc_fused_term(m, n, k,
                                    _ptr(a.data), len(a.views), a_r, a_c, a_co,
                                    _ptr(b.data), len(b.views), b_r, b_c, b_co,
                                    _ptr(c.data), len(c.views), c_r, c_c, c_co,
                                    flags, _ptr(ws), ws.numel(), _stream(), ctypes.byref(st)))
    stats.absorb(st)
    return stats


# ---------------------------------------------------------------- component calls
@dataclass(eq=False)
class PackedBuffer:
    """Sliver-major packed panel in HBM (kernels.py:67-99).

    ``data[s, p, i]``: A side, row ``i`` of sliver ``s`` (width = mr) at depth
    ``p``; B side, column ``i`` (width = nr).  A contiguous float64 CUDA tensor
    (256-byte aligned by the allocator; the reference aligns to a cache line).
    """

    data: object
    width: int
    depth: int

    @property
    def n_slivers(self) -> int:
        return self.data.shape[0]

    def element(self, s: int, p: int, i: int) -> float:
        return float(self.data[s, p, i])

    @classmethod
    def _panel(cls, extent: int, depth: int, width: int, device) -> "PackedBuffer":
        torch = _torch()
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        return cls(torch.zeros((-(-extent // width), depth, width), dtype=torch.float64, device=dev), width, depth)

    @classmethod
    def a_panel(cls, params: BlockingParams, m: int | None = None, k: int | None = None, device=None):
        return cls._panel(params.mc if m is None else min(params.mc, m),
                          params.kc if k is None else min(params.kc, k), params.mr, device)

    @classmethod
    def b_panel(cls, params: BlockingParams, n: int | None = None, k: int | None = None, device=None):
        return cls._panel(params.nc if n is None else min(params.nc, n),
                          params.kc if k is None else min(params.kc, k), params.nr, device)


def _interval(name: str, rng, limit: int, cap: int, align: int):
    lo, hi = rng
    if not 0 <= lo < hi <= limit:
        raise ValueError(f"{name} interval [{lo},{hi}) out of bounds for size {limit}")
    if hi - lo > cap:
        raise ValueError(f"{name} interval [{lo},{hi}) exceeds cache block {cap}")
    if lo % align:
        raise ValueError(f"{name} interval must start at a multiple of {align}")
    return lo, hi


def _pack(which: int, side: OperandTermSide, x_rng, k_rng, width: int, kblock: int, out: PackedBuffer,
          stats: RunStats | None, force_slow: bool) -> None:
    torch = _torch()
    (x0, x1), (k0, k1) = x_rng, k_rng
    if out.width != width or out.depth < k1 - k0 or out.n_slivers < -(-(x1 - x0) // width):
        raise ValueError("packed buffer too small for the requested block")
    if not (isinstance(out.data, torch.Tensor) and out.data.is_cuda and out.data.is_contiguous()
            and out.data.dtype == torch.float64):
        raise ValueError("packed buffer must be a contiguous float64 CUDA tensor (PackedBuffer.a_panel / b_panel)")
    if out.data.device != side.data.device:
        raise ValueError(f"packed buffer on {out.data.device} but the views' parent on {side.data.device}")
    tabs = [_ptr_array([f(v) for v in side.views])
            for f in (lambda v: v.rscat, lambda v: v.cscat, lambda v: v.rbs, lambda v: v.cbs)]
    co = _coeff_array(side.coeffs)
    st = _lib.Stats()
    with torch.cuda.device(side.data.device):
        _lib.check(_lib.lib().stc_pack_panel(which, _ptr(side.data), len(side.views), tabs[0][0], tabs[1][0],
                                             tabs[2][0], tabs[3][0], co, x0, x1 - x0, k0, k1 - k0, width, kblock,
                                             _lib.FLAG_FORCE_SLOW if force_slow else 0, _ptr(out.data), out.depth,
                                             _stream(), ctypes.byref(st)))
    if stats is not None:
        stats.fast_blocks += st.fast_blocks
        stats.slow_blocks += st.slow_blocks


def pack_a(side: OperandTermSide, row_block, k_block, params: BlockingParams, out: PackedBuffer,
           stats: RunStats | None, force_slow: bool = False) -> None:
    """The A-side term sum over row_block x k_block into mr-row slivers (kernels.py:166-182):
    the Strassen packing pass on its own (``stc_pack_panel``), bitwise the reference's panel."""
    if (side.rb, side.cb) != (params.mr, params.kr):
        raise ValueError(f"A-side views need block geometry ({params.mr},{params.kr}), got ({side.rb},{side.cb})")
    rows = _interval("row", row_block, side.m, params.mc, params.mr)
    ks = _interval("k", k_block, side.n, params.kc, params.kr)
    _pack(0, side, rows, ks, params.mr, params.kr, out, stats, force_slow)


def pack_b(side: OperandTermSide, k_block, col_block, params: BlockingParams, out: PackedBuffer,
           stats: RunStats | None, force_slow: bool = False) -> None:
    """The B-side term sum over k_block x col_block into nr-column slivers (kernels.py:185-201)."""
    if (side.rb, side.cb) != (params.kr, params.nr):
        raise ValueError(f"B-side views need block geometry ({params.kr},{params.nr}), got ({side.rb},{side.cb})")
    ks = _interval("k", k_block, side.m, params.kc, params.kr)
    cols = _interval("col", col_block, side.n, params.nc, params.nr)
    _pack(1, side, cols, ks, params.nr, params.kr, out, stats, force_slow)


def microkernel(a_sliver, b_sliver, k: int, targets, stats: RunStats | None, force_slow: bool = False) -> None:
    """One mr x nr tile product, then coeff * tile added into every target (kernels.py:204-233).

    ``a_sliver`` (mr, >= k) and ``b_sliver`` (>= k, nr): numpy arrays or torch tensors;
    ``targets``: ``(view, i0, j0, coeff)`` tuples over device views.  The tile is
    accumulated in the reference's order and roundings (``stc_microtile``: bitwise equal).
    """
    if k == 0:
        return
    torch = _torch()
    targets = list(targets)
    dev = (targets[0][0].base.data.device if targets
           else a_sliver.device if isinstance(a_sliver, torch.Tensor) and a_sliver.is_cuda
           else torch.device("cuda", torch.cuda.current_device()))

    def sliver(x):
        x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)) if isinstance(x, np.ndarray) else x
        if x.dim() != 2:
            raise ValueError("slivers must be 2-D")
        return x.to(device=dev, dtype=torch.float64).contiguous()

    a, b = sliver(a_sliver), sliver(b_sliver)
    mr, nr = a.shape[0], b.shape[1]
    if a.shape[1] < k or b.shape[0] < k:
        raise ValueError("slivers shorter than the requested accumulation depth")
    for view, i0, j0, _ in targets:
        if view.rb != mr or view.cb != nr:
            raise ValueError(f"target blocks ({view.rb},{view.cb}) do not match tile ({mr},{nr})")
        if i0 % mr or j0 % nr:
            raise ValueError("tile origin must be block-aligned")
        if view.base.data is not targets[0][0].base.data:
            raise ValueError("targets of one tile must share one parent tensor")
    if not targets:
        return
    views = [t[0] for t in targets]
    tabs = [_ptr_array([f(v) for v in views])
            for f in (lambda v: v.rscat, lambda v: v.cscat, lambda v: v.rbs, lambda v: v.cbs)]
    co = _coeff_array([t[3] for t in targets])
    i64s = lambda xs: (ctypes.c_int64 * len(xs))(*[int(x) for x in xs])
    st = _lib.Stats()
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().stc_microtile(_ptr(a), a.stride(0), _ptr(b), b.stride(0), int(k), mr, nr,
                                            _ptr(views[0].base.data), len(targets), tabs[0][0], tabs[1][0],
                                            tabs[2][0], tabs[3][0], co, i64s([t[1] for t in targets]),
                                            i64s([t[2] for t in targets]), i64s([v.m for v in views]),
                                            i64s([v.n for v in views]), _lib.FLAG_FORCE_SLOW if force_slow else 0,
                                            _stream(), ctypes.byref(st)))
    if stats is not None:
        stats.fast_updates += st.fast_updates
        stats.slow_updates += st.slow_updates


def _col_major_tensor(mat, name: str) -> DenseTensor:
    torch = _torch()
    if not isinstance(mat, torch.Tensor) or mat.dim() != 2 or mat.dtype != torch.float64:
        raise ValueError(f"{name} must be a 2-D float64 array")
    if mat.shape[0] > 1 and mat.stride(0) != 1 or (mat.shape[1] > 1 and mat.stride(1) != mat.shape[0]):
        raise ValueError(f"{name} must be column-major (order='F')")
    return DenseTensor.from_torch(mat)


def run_gemm_dense(c, a, b, params: BlockingParams = DEFAULT_BLOCKING, stats: RunStats | None = None,
                   threads: int = 1, force_slow: bool = False, workspace=None) -> RunStats:
    """C += A @ B on column-major CUDA matrices through the fused kernel (driver.py:139-152)."""
    m, k = a.shape
    n = b.shape[1]
    if b.shape[0] != k or tuple(c.shape) != (m, n):
        raise ValueError(f"shape mismatch: C{tuple(c.shape)} += A{tuple(a.shape)} @ B{tuple(b.shape)}")
    prim = FusedPrimitive(
        OperandTermSide([matrix_view(_col_major_tensor(a, "a"), params.mr, params.kr)], [1]),
        OperandTermSide([matrix_view(_col_major_tensor(b, "b"), params.kr, params.nr)], [1]),
        OperandTermSide([matrix_view(_col_major_tensor(c, "c"), params.mr, params.nr)], [1]),
    )
    return run_fused(prim, params, stats, threads=threads, force_slow=force_slow)


def _as_device_matrix(mat, device):
    torch = _torch()
    if isinstance(mat, np.ndarray):
        mat = torch.from_numpy(np.asarray(mat, dtype=np.float64)).to(device)
    if mat.dtype != torch.float64 or mat.dim() != 2:
        raise ValueError("matrix must be a 2-D float64 array")
    if not (mat.stride(0) == 1 and (mat.shape[1] <= 1 or mat.stride(1) >= max(mat.shape[0], 1))):
        mat = mat.t().contiguous().t()  # column-major copy
    return mat


def accumulate_dense_to_view(mat, coeff: int, target: BlockScatterView, stats: RunStats,
                             force_slow: bool = False) -> None:
    """target += coeff * mat through the scatter offsets (kernels.py:236-247)."""
    torch = _torch()
    if tuple(mat.shape) != (target.m, target.n):
        raise ValueError(f"matrix shape {tuple(mat.shape)} does not match view {target.m}x{target.n}")
    dev = target.base.data.device
    mat = _as_device_matrix(mat, dev)
    ld = max(mat.stride(1), target.m) if target.n > 1 else max(target.m, 1)
    st = _lib.Stats()
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().stc_accumulate_dense(_ptr(mat), ld, target.m, target.n, _ptr(target.base.data),
                                                   _ptr(target.rscat), _ptr(target.cscat), float(coeff),
                                                   _stream(), ctypes.byref(st)))
    if stats is not None:
        stats.absorb(st)


def unpack_to_dense(side: OperandTermSide, out=None, stats: RunStats | None = None, force_slow: bool = False):
    """Dense column-major sum of the side's views, PAD reads 0 (kernels.py:250-264)."""
    torch = _torch()
    dev = side.data.device
    if out is None:
        out = torch.empty((side.n, side.m), dtype=torch.float64, device=dev).t()
    elif (tuple(out.shape) != (side.m, side.n) or out.dtype != torch.float64 or out.stride(0) != 1
          or (side.n > 1 and out.stride(1) < side.m)):
        raise ValueError(f"out must be a float64 {side.m}x{side.n} matrix")
    ld = out.stride(1) if side.n > 1 else max(side.m, 1)
    pr, ar = _ptr_array([v.rscat for v in side.views])
    pc, ac = _ptr_array([v.cscat for v in side.views])
    co = _coeff_array(side.coeffs)
    st = _lib.Stats()
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().stc_unpack_sum(_ptr(out), ld, side.m, side.n, _ptr(side.data), len(side.views),
                                             pr, pc, co, _stream(), ctypes.byref(st)))
    if stats is not None:
        stats.absorb(st)
    return out


def relative_error(t, t_ref) -> float:
    """||t - t_ref||_F / ||t_ref||_F over every multi-index (oracle.py:110-124).

    Both tensors on the device: reduced there (deterministic order).  Both on
    the host: exactly rounded sums (math.fsum).  0/0 -> 0.0, x/0 -> inf.
    """
    if isinstance(t, DenseTensor) is False or isinstance(t_ref, DenseTensor) is False:
        t = t if isinstance(t, DenseTensor) else DenseTensor.from_torch(t)
        t_ref = t_ref if isinstance(t_ref, DenseTensor) else DenseTensor.from_torch(t_ref)
    if t.extents != t_ref.extents:
        raise ValueError(f"extent mismatch: {t.extents} vs {t_ref.extents}")
    if t.on_device and t_ref.on_device:
        torch = _torch()
        nd = t.ndim
        ext = (ctypes.c_int64 * max(nd, 1))(*t.extents)
        xs = (ctypes.c_int64 * max(nd, 1))(*t.strides)
        rs = (ctypes.c_int64 * max(nd, 1))(*t_ref.strides)
        out = (ctypes.c_double * 2)()
        with torch.cuda.device(t.data.device):
            _lib.check(_lib.lib().stc_sq_norms(nd, ext, _ptr(t.data), xs, t.base_offset, _ptr(t_ref.data), rs,
                                               t_ref.base_offset, out, _stream()))
        num, den = math.sqrt(out[0]), math.sqrt(out[1])
    else:
        a, r = t.to_host(), t_ref.to_host()

        def offs(x):
            o = np.full(1, x.base_offset, dtype=np.int64)
            for e, s in zip(x.extents, x.strides):
                o = (o[:, None] + (np.arange(e, dtype=np.int64) * s)[None, :]).ravel(order="F")
            return o

        va, vr = a.data[offs(a)], r.data[offs(r)]
        num = math.sqrt(math.fsum((va - vr) ** 2))
        den = math.sqrt(math.fsum(vr ** 2))
    if den == 0.0:
        return 0.0 if num == 0.0 else math.inf
    return num / den
