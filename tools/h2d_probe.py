"""H2D bandwidth from pinned host memory: one stream vs two / four concurrent streams
(each copying an equal part), 402 MB total (cfg2's A + B + C)."""
import torch

n = 402653184 // 8
x = torch.empty(n, dtype=torch.float64).pin_memory()
y = torch.empty(n, dtype=torch.float64, device="cuda")
for parts in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(parts)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(4):
        torch.cuda.synchronize()
        e0.record()
        for i, s in enumerate(ss):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                lo, hi = n * i // parts, n * (i + 1) // parts
                y[lo:hi].copy_(x[lo:hi], non_blocking=True)
        for s in ss:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"H2D 402 MB in {parts} stream(s): {best:.3f} ms  {402653184 / best / 1e6:.1f} GB/s")
