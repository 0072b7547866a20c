"""Run statistics and the effective-GFLOPS metric (oracle.py:22-50 in the reference)."""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["RunStats", "effective_gflops"]


@dataclass
class RunStats:
    """Timing and counters of one ``contract`` call.

    ``seconds`` is the wall clock of the whole call, as the reference times it
    (perf_counter around the call body, strassen.py:154,205): planning, host
    staging and transfers for host operands, and the device work, synchronised
    before return.  ``device_seconds`` is the device time of the work the call
    enqueued (CUDA events on its stream).  ``synchronize=False`` calls return
    without either (the caller times its stream).
    ``total_flops`` counts executed MMA flops including tile padding;
    ``effective_gflops`` always uses the classical 2*N_I*N_J*N_P over
    ``seconds``, so Strassen's saving shows as a higher effective rate (same
    definition as the reference, oracle.py:46-50).  Block/update counters are
    per GPU tile (the reference counts per mr x nr register block): fast blocks
    are operand tiles staged by TMA boxes, slow blocks by per-element gathers;
    fast updates are C-tile updates by TMA reduce-add boxes, slow updates by the
    scatter epilogue or the dense-M accumulate pass.  ``leaf_multiplies`` is 7^L
    per contraction as in the reference; ``pieces`` > 1 when host operands were
    contracted in independent pieces (pieces x 7^L leaf products ran).
    """

    seconds: float = 0.0
    total_flops: float = 0.0
    effective_gflops: float = 0.0
    rel_error: float | None = None
    fast_blocks: int = 0
    slow_blocks: int = 0
    fast_updates: int = 0
    slow_updates: int = 0
    leaf_multiplies: int = 0
    work_items: int = 0
    kernel_launches: int = 0
    pieces: int = 1
    device_seconds: float = 0.0

    def total_gflops(self) -> float:
        return self.total_flops / self.seconds / 1e9 if self.seconds > 0 else 0.0

    def absorb(self, st) -> None:
        """Add a C-ABI stc_stats into these counters."""
        self.total_flops += st.total_flops
        self.fast_blocks += st.fast_blocks
        self.slow_blocks += st.slow_blocks
        self.fast_updates += st.fast_updates
        self.slow_updates += st.slow_updates
        self.leaf_multiplies += st.leaf_multiplies
        self.work_items += st.work_items
        self.kernel_launches += st.kernel_launches
        self.pieces = max(1, int(st.pieces))


def effective_gflops(n_i: int, n_j: int, n_p: int, seconds: float) -> float:
    """2 * N_I * N_J * N_P / seconds / 1e9."""
    if seconds <= 0:
        raise ValueError(f"seconds must be positive, got {seconds}")
    return 2.0 * n_i * n_j * n_p / seconds / 1e9
