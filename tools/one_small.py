import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1704_03092_b200 as stc
spec = stc.parse_benchmark_line("abij abef efij & a:24;b:24;i:24;j:24;e:24;f:24;")
def rm(ext):
    out, run = [], 1
    for e in reversed(ext): out.append(run); run *= e
    return tuple(reversed(out))
ext = (24, 24, 24, 24)
a = stc.DenseTensor(ext, rm(ext), np.random.default_rng(7).uniform(-1, 1, 24**4)).to_device()
b = stc.DenseTensor(ext, rm(ext), np.random.default_rng(8).uniform(-1, 1, 24**4)).to_device()
c = stc.DenseTensor(ext, rm(ext), np.zeros(24**4)).to_device()
stc.contract(spec, a, b, c, 0, "abc", force_slow=True)
print("done")
