"""Does a PCIe copy on another stream slow the fused kernel?  Device-resident cfg2 L2 ABC
timed alone, under a concurrent 1.2 GB pinned H2D copy, under a D2H copy, and as two
concurrent contractions on two streams."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
import numpy as np, torch
import paper_1704_03092_b200 as stc
from perf_probe import CONFIGS, dev_tensor

spec = stc.parse_benchmark_line(CONFIGS["cfg2"][0])
a = dev_tensor(spec.tensor_extents(spec.labels_a), 1)
b = dev_tensor(spec.tensor_extents(spec.labels_b), 2)
c = dev_tensor(spec.tensor_extents(spec.labels_c), 3, zero=True)
c2 = dev_tensor(spec.tensor_extents(spec.labels_c), 4, zero=True)
hx = torch.zeros(150 * 2 ** 20, dtype=torch.float64).pin_memory()
dx = torch.empty_like(hx, device="cuda")
side = torch.cuda.Stream()
s2 = torch.cuda.Stream()


def run(label, copy=None, twin=False):
    for _ in range(2):
        stc.contract(spec, a, b, c, 2, "abc")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ce0, ce1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if copy:
        with torch.cuda.stream(side):
            ce0.record()
            (dx.copy_(hx, non_blocking=True) if copy == "h2d" else hx.copy_(dx, non_blocking=True))
            ce1.record()
    e0.record()
    if twin:
        s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s2):
            stc.contract(spec, a, b, c2, 2, "abc", synchronize=False)
    stc.contract(spec, a, b, c, 2, "abc", synchronize=False)
    if twin:
        torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    extra = f"  copy {ce0.elapsed_time(ce1):.2f} ms" if copy else ""
    print(f"{label:28s} contract {e0.elapsed_time(e1):.3f} ms{extra}", flush=True)


for _ in range(2):
    run("alone")
    run("with H2D 1.2 GB", "h2d")
    run("with D2H 1.2 GB", "d2h")
    run("two concurrent (2 streams)", twin=True)
