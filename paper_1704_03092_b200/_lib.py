"""ctypes binding of libstc_b200.so (the C ABI declared in include/stc_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1704_03092_b200/csrc``).  There is no fallback: if the library
is missing or CUDA is unavailable, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import pathlib

__all__ = ["lib", "Bundle", "Problem", "Stats", "PlanInfo", "check", "MAX_LABELS", "PAD", "LIB_PATH"]

LIB_PATH = pathlib.Path(os.environ.get("STC_LIBRARY", pathlib.Path(__file__).resolve().parent / "libstc_b200.so"))
MAX_LABELS = 16
PAD = -(1 << 63)

STC_OK, STC_EINVAL, STC_ECAP, STC_ECUDA, STC_EWORKSPACE, STC_EOVERLAP = range(6)
FLAG_FORCE_SLOW, FLAG_VALIDATE, FLAG_REFERENCE_TILING = 1, 2, 4
VARIANT_CODES = {"abc": 0, "ab": 1, "naive": 2}


class Bundle(ctypes.Structure):
    _fields_ = [("nlab", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("ext", ctypes.c_int64 * MAX_LABELS), ("str", ctypes.c_int64 * MAX_LABELS)]

    @classmethod
    def of(cls, extents, strides) -> "Bundle":
        b = cls()
        if len(extents) > MAX_LABELS:
            raise ValueError(f"bundles are limited to {MAX_LABELS} labels")
        b.nlab = len(extents)
        for d, (e, s) in enumerate(zip(extents, strides)):
            b.ext[d] = int(e)
            b.str[d] = int(s)
        return b


class Problem(ctypes.Structure):
    _fields_ = [("a_row", Bundle), ("a_col", Bundle), ("b_row", Bundle), ("b_col", Bundle),
                ("c_row", Bundle), ("c_col", Bundle),
                ("a_base", ctypes.c_int64), ("b_base", ctypes.c_int64), ("c_base", ctypes.c_int64),
                ("level", ctypes.c_int32), ("variant", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("tiling", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [("total_flops", ctypes.c_double), ("fast_blocks", ctypes.c_int64),
                ("slow_blocks", ctypes.c_int64), ("fast_updates", ctypes.c_int64),
                ("slow_updates", ctypes.c_int64), ("leaf_multiplies", ctypes.c_int64),
                ("work_items", ctypes.c_int64), ("kernel_launches", ctypes.c_int64), ("pieces", ctypes.c_int64)]


class PlanInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("ticketed", "presum", "need_pack", "tshape", "fused_direct", "c_boxes",
                                              "batch", "nbatches", "terms", "presum_sides")] + \
               [(n, ctypes.c_int64) for n in ("tiles", "mq_pad", "nq_pad", "kq_pad")] + [("workspace", ctypes.c_size_t)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_ if n != "_pad"}


_EXPORTS = (
    "stc_last_error", "stc_abi_version", "stc_workspace_size", "stc_contract", "stc_bundle_scatter",
    "stc_block_vector", "stc_fused_term_workspace_size", "stc_fused_term", "stc_accumulate_dense",
    "stc_unpack_sum", "stc_pack_panel", "stc_microtile", "stc_sq_norms", "stc_set_kernel_events", "stc_set_c_ready",
    "stc_host_workspace_size", "stc_contract_host", "stc_host_plan", "stc_fill_uniform", "stc_plan_describe",
    "stc_shard_problem", "stc_host_grid", "stc_sharded_workspace_size", "stc_contract_sharded",
)

_lib = None


def _declare(l):
    P = ctypes.POINTER
    vp, i64, i32, u32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_size_t
    pp = P(ctypes.c_void_p)
    dp = P(ctypes.c_double)
    l.stc_last_error.restype = ctypes.c_char_p
    l.stc_abi_version.restype = ctypes.c_int
    l.stc_workspace_size.argtypes = [P(Problem), P(sz)]
    l.stc_contract.argtypes = [P(Problem), vp, vp, vp, vp, sz, vp, P(Stats)]
    l.stc_bundle_scatter.argtypes = [P(Bundle), i64, i64, vp, vp]
    l.stc_block_vector.argtypes = [vp, i64, i64, i64, vp, vp]
    l.stc_fused_term_workspace_size.argtypes = [i64, i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, P(sz)]
    l.stc_fused_term.argtypes = [i64, i64, i64,
                                 vp, ctypes.c_int, pp, pp, dp,
                                 vp, ctypes.c_int, pp, pp, dp,
                                 vp, ctypes.c_int, pp, pp, dp,
                                 u32, vp, sz, vp, P(Stats)]
    l.stc_accumulate_dense.argtypes = [vp, i64, i64, i64, vp, vp, vp, ctypes.c_double, vp, P(Stats)]
    l.stc_unpack_sum.argtypes = [vp, i64, i64, i64, vp, ctypes.c_int, pp, pp, dp, vp, P(Stats)]
    l.stc_pack_panel.argtypes = [ctypes.c_int, vp, ctypes.c_int, pp, pp, pp, pp, dp, i64, i64, i64, i64, i64, i64, u32,
                                 vp, i64, vp, P(Stats)]
    l.stc_microtile.argtypes = [vp, i64, vp, i64, i64, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int, pp, pp, pp, pp,
                                dp, P(i64), P(i64), P(i64), P(i64), u32, vp, P(Stats)]
    l.stc_sq_norms.argtypes = [ctypes.c_int, P(i64), vp, P(i64), i64, vp, P(i64), i64, dp, vp]
    l.stc_set_kernel_events.argtypes = [vp, vp]
    l.stc_set_c_ready.argtypes = [vp]
    l.stc_host_workspace_size.argtypes = [P(Problem), P(sz)]
    l.stc_contract_host.argtypes = [P(Problem), vp, vp, vp, vp, vp, vp, vp, sz, vp, P(Stats)]
    l.stc_host_plan.argtypes = [P(Problem), P(ctypes.c_int32), P(ctypes.c_int32), P(ctypes.c_int32)]
    l.stc_host_grid.argtypes = [P(Problem)] + [P(ctypes.c_int32)] * 4
    l.stc_fill_uniform.argtypes = [vp, ctypes.c_int, P(i64), P(i64), i64, ctypes.c_uint64, vp]
    l.stc_plan_describe.argtypes = [P(Problem), ctypes.c_int, P(PlanInfo)]
    l.stc_shard_problem.argtypes = [P(Problem), ctypes.c_int, ctypes.c_int, ctypes.c_int, P(Problem), P(i64), P(i64),
                                    P(i32)]
    l.stc_sharded_workspace_size.argtypes = [P(Problem), ctypes.c_int, ctypes.c_int, P(sz)]
    l.stc_contract_sharded.argtypes = [P(Problem), ctypes.c_int, P(ctypes.c_int), ctypes.c_int, pp, pp, pp, pp,
                                       P(sz), pp, ctypes.c_int, P(Stats)]
    for name in _EXPORTS:
        if name not in ("stc_last_error",):
            getattr(l, name).restype = ctypes.c_int if name != "stc_last_error" else ctypes.c_char_p


def lib():
    """Load (once) and return the library; raises if it was never built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH.name} is not built; run __graft_entry__.build() or "
                f"`make -C {LIB_PATH.parent / 'csrc'}` (there is no CPU fallback)")
        l = ctypes.CDLL(str(LIB_PATH))
        _declare(l)
        _lib = l
    return _lib


def exported_symbols():
    return _EXPORTS


def check(rc: int) -> None:
    """Map a C-ABI status code to the reference's exception conventions."""
    if rc == STC_OK:
        return
    msg = lib().stc_last_error().decode(errors="replace")
    if rc in (STC_EINVAL, STC_ECAP, STC_EWORKSPACE, STC_EOVERLAP):
        raise ValueError(msg)
    raise RuntimeError(msg)
