"""Where the time of a small contraction goes (cfg1, 576^3): python tools/small_probe.py [level variant]...

Per (level, variant):
  sync    -- contract() device_seconds (events around the call; the host's issue time
             is inside it when the GPU runs dry), best of 20
  stream  -- 200 calls with synchronize=False back to back, events around all of them:
             the per-call device rate when the host issues ahead
  wall    -- perf_counter over the same 200 calls (+ one synchronize): the host's rate
  capi    -- 200 bare stc_contract calls (problem struct and workspace prepared once):
             host time per call of the library alone
"""

import ctypes
import pathlib
import sys
import time

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
import paper_1704_03092_b200 as stc  # noqa: E402
from paper_1704_03092_b200 import _lib  # noqa: E402
from paper_1704_03092_b200.strassen import problem_of  # noqa: E402
from perf_probe import CONFIGS, dev_tensor  # noqa: E402


def main(argv):
    line = CONFIGS["cfg1"][0]
    runs = [(int(argv[i]), argv[i + 1]) for i in range(0, len(argv), 2)] or [(1, "abc"), (2, "abc"), (0, "abc"),
                                                                           (1, "ab")]
    spec = stc.parse_benchmark_line(line)
    a = dev_tensor(spec.tensor_extents(spec.labels_a), 1)
    b = dev_tensor(spec.tensor_extents(spec.labels_b), 2)
    c = dev_tensor(spec.tensor_extents(spec.labels_c), 3, zero=True)
    flop = 2.0 * spec.n_i * spec.n_j * spec.n_p
    n = 200
    for level, variant in runs:
        for _ in range(3):
            stc.contract(spec, a, b, c, level, variant)
        sync = min(stc.contract(spec, a, b, c, level, variant).device_seconds for _ in range(20))
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(s)
        for _ in range(n):
            stc.contract(spec, a, b, c, level, variant, synchronize=False)
        e1.record(s)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        stream = e0.elapsed_time(e1) * 1e-3 / n
        # the bare C ABI
        prob = problem_of(spec, a, b, c, level, stc.Variant(variant), 0)
        L = _lib.lib()
        need = ctypes.c_size_t()
        _lib.check(L.stc_workspace_size(ctypes.byref(prob), ctypes.byref(need)))
        ws = torch.empty(int(need.value), dtype=torch.uint8, device="cuda")
        st = _lib.Stats()
        args = (ctypes.byref(prob), ctypes.c_void_p(a.data.data_ptr()), ctypes.c_void_p(b.data.data_ptr()),
                ctypes.c_void_p(c.data.data_ptr()), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                ctypes.c_void_p(s.cuda_stream), ctypes.byref(st))
        _lib.check(L.stc_contract(*args))
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        e0.record(s)
        for _ in range(n):
            L.stc_contract(*args)
        e1.record(s)
        h1 = time.perf_counter()
        torch.cuda.synchronize()
        capi_dev = e0.elapsed_time(e1) * 1e-3 / n
        print(f"cfg1 L{level} {variant:5s} sync {sync * 1e6:7.1f} us ({flop / sync / 1e12:5.2f} TF/s)  "
              f"stream {stream * 1e6:7.1f} us ({flop / stream / 1e12:5.2f} TF/s)  wall {(t2 - t0) / n * 1e6:7.1f} us "
              f"(issue {(t1 - t0) / n * 1e6:6.1f})  capi host {(h1 - h0) / n * 1e6:6.1f} us dev {capi_dev * 1e6:6.1f} us"
              f"  launches {st.kernel_launches}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
