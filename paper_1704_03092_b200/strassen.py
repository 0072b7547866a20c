"""The drop-in entry point: Strassen tensor contraction on the B200.

``contract(spec, a, b, c, level, variant, ...) -> RunStats`` keeps the
signature, argument meaning and error behaviour of the reference's
``strassen_tc.contract`` (/root/reference/pkg/src/strassen_tc/strassen.py:141-207):

* C += A.B over the bundles of ``spec`` with an L-level Strassen recursion
  (7^L leaf products over 4^L quadrants, PAD-padded to a multiple of 2^L);
* variants ABC (operand sums fused into the DMMA kernel's staging, +/-M fused
  into its epilogue), AB (dense M per term, then accumulate) and NAIVE (dense
  operand sums, dense GEMM, accumulate) -- strassen.py:173-203;
* ``ValueError`` before C is touched for bad extents ("extents") or levels
  above the cap ("cap"), strassen.py:130-134 / 80-81.

Operands may be reference-style ``DenseTensor`` objects with host (numpy)
storage -- staged through HBM, C copied back -- or HBM-resident: strided
float64 CUDA ``torch.Tensor`` or ``DenseTensor`` with CUDA storage.  The work
itself always runs in ``libstc_b200.so`` (C ABI, include/stc_b200.h); there is
no CPU path.  ``params`` is the GPU tile config (``views.TileConfig``: CTA tile
shape, ring depth -- bitwise the same C whatever it is) or the reference's CPU
cache blocking (``BlockingParams``, validated on construction like the
reference's; the planner then chooses); ``threads`` is ignored.
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib
from .stats import RunStats, effective_gflops
from .tensor import ContractionSpec, DenseTensor
from .views import DEFAULT_BLOCKING, BlockingParams, check_c_targets, make_view, quadrant_views, tiling_code

__all__ = ["MAX_LEVEL", "DEVICE_MAX_LEVEL", "StrassenTerm", "Variant", "contract", "strassen_terms",
           "problem_of", "quadrant_rc", "describe_plan"]

MAX_LEVEL = 2          # reference cap without allow_deep (strassen.py:38)
DEVICE_MAX_LEVEL = 4   # 2^L views per side must fit the kernel's op tables


class Variant(Enum):
    ABC = "abc"
    AB = "ab"
    NAIVE = "naive"


@dataclass(frozen=True)
class StrassenTerm:
    """Quadrant ids with +/-1 signs per operand (strassen.py:47-53)."""

    a_ops: tuple
    b_ops: tuple
    c_ops: tuple


# M0..M6 of one Strassen level, quadrants 0=TL 1=TR 2=BL 3=BR (strassen.py:56-65).
_ONE_LEVEL = (
    (((0, 1), (3, 1)), ((0, 1), (3, 1)), ((0, 1), (3, 1))),
    (((2, 1), (3, 1)), ((0, 1),), ((2, 1), (3, -1))),
    (((0, 1),), ((1, 1), (3, -1)), ((1, 1), (3, 1))),
    (((3, 1),), ((2, 1), (0, -1)), ((0, 1), (2, 1))),
    (((0, 1), (1, 1)), ((3, 1),), ((1, 1), (0, -1))),
    (((2, 1), (0, -1)), ((0, 1), (1, 1)), ((3, 1),)),
    (((1, 1), (3, -1)), ((2, 1), (3, 1)), ((0, 1),)),
)


def strassen_terms(level: int, allow_deep: bool = False) -> list:
    """7^L terms over 4^L quadrants; level l substitutes level l-1 into each
    level-1 operand: (q * 4^(l-1) + q2, s * s2), outer level first
    (strassen.py:70-94)."""
    if level < 0:
        raise ValueError(f"level must be non-negative, got {level}")
    if level > MAX_LEVEL and not allow_deep:
        raise ValueError(f"level {level} exceeds the cap of {MAX_LEVEL} (pass allow_deep to override)")
    terms = _TERMS.get(level)
    if terms is None:
        table = [(((0, 1),), ((0, 1),), ((0, 1),))]
        for lev in range(1, level + 1):
            scale = 4 ** (lev - 1)
            table = [
                tuple(tuple((q * scale + q2, s * s2) for q, s in outer[side] for q2, s2 in inner[side])
                      for side in range(3))
                for outer in _ONE_LEVEL
                for inner in table
            ]
        terms = _TERMS[level] = tuple(StrassenTerm(*t) for t in table)  # immutable: built once per level
    return list(terms)


_TERMS: dict = {}


def quadrant_rc(q: int, level: int) -> tuple:
    """Quadrant id -> (row block, col block) in the 2^L x 2^L grid."""
    r = c = 0
    for l in range(level):
        d = (q >> (2 * (level - 1 - l))) & 3
        r, c = 2 * r + (d >> 1), 2 * c + (d & 1)
    return r, c


def _variant(v) -> Variant:
    if isinstance(v, Variant):
        return v
    if hasattr(v, "value"):
        v = v.value
    try:
        return Variant(str(v).lower())
    except ValueError:
        raise ValueError(f"unknown variant {v!r}") from None


def _as_dense(t, name: str) -> DenseTensor:
    if isinstance(t, DenseTensor):
        return t
    if type(t).__module__.startswith("torch"):
        return DenseTensor.from_torch(t)
    if all(hasattr(t, a) for a in ("extents", "strides", "data", "base_offset")):  # reference DenseTensor
        return DenseTensor(t.extents, t.strides, t.data, t.base_offset)
    raise TypeError(f"tensor {name} must be a DenseTensor or a torch.Tensor")


def _check_operands(spec: ContractionSpec, a: DenseTensor, b: DenseTensor, c: DenseTensor) -> None:
    for t, labels, name in ((a, spec.labels_a, "A"), (b, spec.labels_b, "B"), (c, spec.labels_c, "C")):
        want = spec.tensor_extents(labels)
        if tuple(t.extents) != want:
            raise ValueError(f"tensor {name} extents {tuple(t.extents)} do not match spec {want}")


def problem_of(spec: ContractionSpec, a: DenseTensor, b: DenseTensor, c: DenseTensor, level: int,
               variant: Variant, flags: int = 0, tiling: int = 0) -> _lib.Problem:
    """The C-ABI problem descriptor: the six bundles of the three views
    (``tiling``: views.TileConfig.code, 0 for the planner's choice)."""

    def bundle(labels: str, tensor_labels: str, t: DenseTensor) -> _lib.Bundle:
        axes = [tensor_labels.index(l) for l in labels]
        return _lib.Bundle.of([t.extents[x] for x in axes], [t.strides[x] for x in axes])

    p = _lib.Problem()
    p.a_row, p.a_col = bundle(spec.bundle_i, spec.labels_a, a), bundle(spec.bundle_p, spec.labels_a, a)
    p.b_row, p.b_col = bundle(spec.bundle_p, spec.labels_b, b), bundle(spec.bundle_j, spec.labels_b, b)
    p.c_row, p.c_col = bundle(spec.bundle_i, spec.labels_c, c), bundle(spec.bundle_j, spec.labels_c, c)
    p.a_base, p.b_base, p.c_base = a.base_offset, b.base_offset, c.base_offset
    p.level = int(level)
    p.variant = _lib.VARIANT_CODES[variant.value]
    p.flags = int(flags)
    p.tiling = int(tiling)
    return p


# contract()'s per-call host work on a repeated problem (benchmark loops, small
# contractions): the operand check and the C-ABI descriptor are memoised on the
# spec object and the tensors' geometry.  The spec is kept alive by the entry, so
# its id is not reused while cached.
_PROBLEMS: dict = {}


def _geometry(t: DenseTensor) -> tuple:
    return t.extents, t.strides, t.base_offset


def _checked_problem(spec: ContractionSpec, a: DenseTensor, b: DenseTensor, c: DenseTensor, level: int,
                     variant: Variant, flags: int, tiling: int = 0) -> _lib.Problem:
    """_check_operands + problem_of, memoised (the descriptor is shared: read-only)."""
    key = (id(spec), _geometry(a), _geometry(b), _geometry(c), int(level), variant, int(flags), int(tiling))
    hit = _PROBLEMS.get(key)
    if hit is not None and hit[0] is spec:
        return hit[1]
    _check_operands(spec, a, b, c)
    prob = problem_of(spec, a, b, c, level, variant, flags, tiling)
    if len(_PROBLEMS) >= 256:
        _PROBLEMS.clear()
    _PROBLEMS[key] = (spec, prob)
    return prob


def describe_plan(spec: ContractionSpec, a, b, c, level: int, variant, grid: int = 148,
                  force_slow: bool = False, reference_tiling: bool = False,
                  params: BlockingParams = DEFAULT_BLOCKING) -> dict:
    """The execution path the library plans for this contraction (no device
    needed): ticketed / pre-summed / repacked / tile shape / batches / workspace."""
    a, b, c = _as_dense(a, "A"), _as_dense(b, "B"), _as_dense(c, "C")
    _check_operands(spec, a, b, c)
    flags = (_lib.FLAG_FORCE_SLOW if force_slow else 0) | (_lib.FLAG_REFERENCE_TILING if reference_tiling else 0)
    prob = problem_of(spec, a, b, c, level, _variant(variant), flags, tiling_code(params))
    info = _lib.PlanInfo()
    _lib.check(_lib.lib().stc_plan_describe(ctypes.byref(prob), int(grid), ctypes.byref(info)))
    return info.as_dict()


def _validate_targets(spec, c: DenseTensor, level: int, terms) -> None:
    """validate=True: every term's C targets pairwise disjoint (driver.py:53-61)."""
    axes = {lab: i for i, lab in enumerate(spec.labels_c)}
    v = make_view(c, spec.bundle_i, spec.bundle_j, axes, 8, 4)
    quads = {0: v} if level == 0 else quadrant_views(v, level)
    for term in terms:
        check_c_targets([quads[q] for q, _ in term.c_ops])


def _flat_host(t: DenseTensor):
    """(pointer, elements) of a contiguous float64 host storage, else None."""
    import torch

    d = t.data
    if torch.is_tensor(d):
        if d.dtype != torch.float64 or not d.is_contiguous():
            return None
        return d.data_ptr(), d.numel()
    if not isinstance(d, np.ndarray) or d.dtype != np.float64 or not d.flags.c_contiguous or not d.flags.writeable:
        return None
    return d.ctypes.data, d.size


def _contract_host(spec, a, b, c, level, variant, force_slow, reference_tiling, validate, terms, dev,
                   t_start, tiling=0) -> RunStats:
    """Host operands: stc_contract_host pipelines the uploads, the piecewise
    contraction and the download of C (stc_host.cu)."""
    import torch

    (pa, na), (pb, nb), (pc, nc) = _flat_host(a), _flat_host(b), _flat_host(c)
    if validate:  # the check needs C's geometry only: an uninitialised device stand-in
        stand_in = torch.empty(max(nc, 1), dtype=torch.float64, device=dev)
        _validate_targets(spec, DenseTensor(c.extents, c.strides, stand_in, c.base_offset), level, terms)
        del stand_in
    flags = (_lib.FLAG_FORCE_SLOW if force_slow else 0) | (_lib.FLAG_REFERENCE_TILING if reference_tiling else 0)
    prob = problem_of(spec, a, b, c, level, variant, flags, tiling)
    L = _lib.lib()
    stats = RunStats()
    with torch.cuda.device(dev):
        need = ctypes.c_size_t()
        _lib.check(L.stc_host_workspace_size(ctypes.byref(prob), ctypes.byref(need)))
        ws = torch.empty(max(int(need.value), 256), dtype=torch.uint8, device=dev)
        da, db, dc = (torch.empty(max(n, 1), dtype=torch.float64, device=dev) for n in (na, nb, nc))
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st = _lib.Stats()
        e0.record(stream)
        _lib.check(L.stc_contract_host(ctypes.byref(prob), ctypes.c_void_p(pa), ctypes.c_void_p(pb),
                                       ctypes.c_void_p(pc), ctypes.c_void_p(da.data_ptr()),
                                       ctypes.c_void_p(db.data_ptr()), ctypes.c_void_p(dc.data_ptr()),
                                       ctypes.c_void_p(ws.data_ptr()), ws.numel(), ctypes.c_void_p(stream.cuda_stream),
                                       ctypes.byref(st)))
        e1.record(stream)
        e1.synchronize()  # C is host memory: complete before returning
        stats.absorb(st)
        stats.device_seconds = max(e0.elapsed_time(e1) * 1e-3, 1e-12)
    stats.seconds = max(time.perf_counter() - t_start, 1e-12)
    stats.effective_gflops = effective_gflops(spec.n_i, spec.n_j, spec.n_p, stats.seconds)
    return stats


_SIDE = {}
_ONE = []
_WS = {}
_WS_KEEP = 64 << 20  # workspaces up to this size stay cached per (device, stream)


def _workspace(dev, stream, nbytes: int):
    """The call's workspace.  Small ones are kept per (device, stream) and reused by
    the next call on that stream (stream order serialises the uses; the pointer then
    stays stable, which the library's graph replay keys on); large ones come from
    the caching allocator each call and are released after it."""
    import torch

    if nbytes > _WS_KEEP:
        return torch.empty(nbytes, dtype=torch.uint8, device=dev)
    key = (dev.index, stream.cuda_stream)
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = _WS[key] = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=dev)
    return ws


def _pinned_one():
    """A page-locked int32 1 (source of the c_ready flag copy)."""
    import torch

    if not _ONE:
        _ONE.append(torch.ones(1, dtype=torch.int32).pin_memory())
    return _ONE[0]


def _side_stream(dev):
    """One upload stream per device, reused across calls."""
    import torch

    key = dev.index
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(device=dev)
    return _SIDE[key]


def contract(spec: ContractionSpec, a, b, c, level: int, variant, params: BlockingParams = DEFAULT_BLOCKING,
             threads: int = 1, force_slow: bool = False, allow_deep: bool = False, validate: bool = False,
             reference_tiling: bool = False, kernel_events=None, synchronize: bool = True) -> RunStats:
    """C += contraction of A and B with an L-level Strassen recursion on the B200.

    Level 0 is the plain block-scatter GEMM.  All variants compute the same
    result up to floating-point reordering and execute exactly 7^level leaf
    products.  ``RunStats.seconds`` is the wall clock of the whole call (the
    reference's timer, strassen.py:154,205); ``device_seconds`` the CUDA-event
    time of the work it enqueued on the current stream.  ``params``: a
    ``views.TileConfig`` (the GPU tile config that replaces the reference's
    blocking: CTA tile shape, ring depth; bitwise the same C) or the reference's
    ``BlockingParams`` (CPU cache blocking, validated like the reference does;
    the planner chooses the tiles).  ``threads`` is ignored.
    """
    t_start = time.perf_counter()
    tiling = tiling_code(params)
    a, b, c = _as_dense(a, "A"), _as_dense(b, "B"), _as_dense(c, "C")
    flags = (_lib.FLAG_FORCE_SLOW if force_slow else 0) | (_lib.FLAG_REFERENCE_TILING if reference_tiling else 0)
    try:
        known = _variant(variant)
    except ValueError:
        known = None
    # the operand check (memoised with the descriptor), then the level, then the variant
    prob = _checked_problem(spec, a, b, c, level, known, flags, tiling) if known is not None else None
    if prob is None:
        _check_operands(spec, a, b, c)
    terms = strassen_terms(level, allow_deep)
    if level > DEVICE_MAX_LEVEL:
        raise ValueError(f"level {level} exceeds the device cap of {DEVICE_MAX_LEVEL}")
    variant = _variant(variant)
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 contraction path has no CPU fallback")
    dev = next((t.data.device for t in (c, a, b) if t.on_device), torch.device("cuda", torch.cuda.current_device()))
    # All operands in host memory (contiguous float64 storage): stc_contract_host
    # pipelines the uploads, the piecewise contraction and the download of C
    # (STC_HOST_PIPELINE=0 disables it).  Otherwise host operands are staged
    # through HBM; opt-in (STC_C_OVERLAP=1) a host C is uploaded on a side stream
    # under the DMMA main loop, the kernels waiting on the device for its ready
    # flag before their first C update (stc_set_c_ready).
    if not (a.on_device or b.on_device or c.on_device) and kernel_events is None \
            and os.environ.get("STC_HOST_PIPELINE", "1") != "0" and all(_flat_host(t) is not None for t in (a, b, c)):
        return _contract_host(spec, a, b, c, level, variant, force_slow, reference_tiling, validate, terms, dev,
                              t_start, tiling)
    c_ready = None
    A = a if a.on_device else a.to_device(dev)
    B = b if b.on_device else b.to_device(dev)
    if not c.on_device and os.environ.get("STC_C_OVERLAP", "0") != "0":
        # C's upload starts after A and B's (it would only slow them down) and runs
        # under the DMMA main loop; buffers come from the main stream's pool
        main = torch.cuda.current_stream(dev)
        c_ready = torch.zeros(1, dtype=torch.int32, device=dev)
        src = c.data if torch.is_tensor(c.data) else torch.from_numpy(c.data)
        cd = torch.empty(src.shape, dtype=src.dtype, device=dev)
        side = _side_stream(dev)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            cd.copy_(src, non_blocking=src.is_pinned())
            # by the copy engine, not a fill kernel: the contraction's persistent CTAs
            # occupy every SM while they spin on this flag
            c_ready.copy_(_pinned_one(), non_blocking=True)
        C = DenseTensor(c.extents, c.strides, cd, c.base_offset)
    else:
        C = c if c.on_device else c.to_device(dev)
    if validate:
        _validate_targets(spec, C, level, terms)
    L = _lib.lib()
    stats = RunStats()
    timed = not (c.on_device and not synchronize)  # stream-ordered calls: no events
    with torch.cuda.device(dev):
        need = ctypes.c_size_t()
        _lib.check(L.stc_workspace_size(ctypes.byref(prob), ctypes.byref(need)))
        stream = torch.cuda.current_stream()
        ws = _workspace(dev, stream, max(int(need.value), 256))
        if os.environ.get("STC_DEBUG_POISON"):  # debugging aid: the library must not read stale workspace
            ws.fill_(int(os.environ["STC_DEBUG_POISON"]) & 255)
        e0, e1 = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) if timed else (None, None)
        st = _lib.Stats()
        if kernel_events is not None:  # profiling hook: events around the DMMA launch(es)
            L.stc_set_kernel_events(ctypes.c_void_p(kernel_events[0].cuda_event),
                                    ctypes.c_void_p(kernel_events[1].cuda_event))
        if c_ready is not None:
            L.stc_set_c_ready(ctypes.c_void_p(c_ready.data_ptr()))
        if timed:
            e0.record(stream)
        _lib.check(L.stc_contract(ctypes.byref(prob), ctypes.c_void_p(A.data.data_ptr()),
                                  ctypes.c_void_p(B.data.data_ptr()), ctypes.c_void_p(C.data.data_ptr()),
                                  ctypes.c_void_p(ws.data_ptr()), ws.numel(), ctypes.c_void_p(stream.cuda_stream),
                                  ctypes.byref(st)))
        if timed:
            e1.record(stream)
        stats.absorb(st)
        if not c.on_device:
            if c_ready is not None:
                stream.wait_stream(side)  # C's upload is complete before it is read back
            c.store_from(C)  # synchronous download of C (host operands)
        elif not synchronize:
            # stream-ordered only: the caller times the stream itself; no per-call seconds
            return stats
        e1.synchronize()
        stats.device_seconds = max(e0.elapsed_time(e1) * 1e-3, 1e-12)
    stats.seconds = max(time.perf_counter() - t_start, 1e-12)
    stats.effective_gflops = effective_gflops(spec.n_i, spec.n_j, spec.n_p, stats.seconds)
    return stats


def contract_reference(spec: ContractionSpec, a, b, c) -> None:
    """C += the classical contraction (the reference's ``contract_reference``, oracle.py:82-94).

    The reference loops every (I, J, P) multi-index on the CPU; here it is the
    level-0 contraction on the DMMA kernel in the reference's tile order -- the
    same products, summed over P in the kernel's k order (differences at
    rounding level, exact on integer data).  Not the test oracle: the tests
    check against ``oracle/`` on the CPU.
    """
    contract(spec, a, b, c, 0, Variant.ABC, reference_tiling=True)

