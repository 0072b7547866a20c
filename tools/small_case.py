"""One small irregular contraction (for compute-sanitizer): python tools/small_case.py level variant"""
import pathlib
import sys

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
import paper_1704_03092_b200 as stc  # noqa: E402
from perf_probe import dev_tensor  # noqa: E402

level, variant = int(sys.argv[1]), sys.argv[2]
line = sys.argv[3] if len(sys.argv) > 3 else "abcij eafbc ifje & a:10;b:7;c:13;i:14;j:9;e:18;f:11;"
spec = stc.parse_benchmark_line(line)
a = dev_tensor(spec.tensor_extents(spec.labels_a), 1)
b = dev_tensor(spec.tensor_extents(spec.labels_b), 2)
c = dev_tensor(spec.tensor_extents(spec.labels_c), 3)
stc.contract(spec, a, b, c, level, variant)
torch.cuda.synchronize()
print("done")
