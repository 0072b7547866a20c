"""Per-kernel device timeline of repeated warm contract() calls (CUPTI through torch.profiler).

python tools/kernel_timeline.py cfg1 1 abc [calls]
Prints, per kernel name: count, mean duration, and the mean gap before it (from the
previous kernel's end on the device), then the mean span of one call.
"""

import collections
import pathlib
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
import paper_1704_03092_b200 as stc  # noqa: E402
from perf_probe import CONFIGS, dev_tensor  # noqa: E402


def main(argv):
    name, level, variant = argv[0], int(argv[1]), argv[2]
    calls = int(argv[3]) if len(argv) > 3 else 50
    spec = stc.parse_benchmark_line(CONFIGS[name][0])
    a = dev_tensor(spec.tensor_extents(spec.labels_a), 1)
    b = dev_tensor(spec.tensor_extents(spec.labels_b), 2)
    c = dev_tensor(spec.tensor_extents(spec.labels_c), 3, zero=True)
    for _ in range(5):
        stc.contract(spec, a, b, c, level, variant)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(calls):
            stc.contract(spec, a, b, c, level, variant, synchronize=False)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    dur = collections.defaultdict(list)
    gap = collections.defaultdict(list)
    prev_end = None
    for e in evs:
        key = e.name.split("(")[0][:60]
        dur[key].append(e.time_range.end - e.time_range.start)
        if prev_end is not None:
            gap[key].append(e.time_range.start - prev_end)
        prev_end = e.time_range.end
    print(f"{name} L{level} {variant}: {len(evs)} device ops over {calls} calls")
    for k, v in dur.items():
        g = gap.get(k, [0])
        print(f"  {k:60s} n={len(v):4d}  mean {sum(v) / len(v):8.2f} us  gap before {sum(g) / len(g):7.2f} us")
    span = (evs[-1].time_range.end - evs[0].time_range.start) / calls
    print(f"  per call span {span:.2f} us")


if __name__ == "__main__":
    main(sys.argv[1:])
