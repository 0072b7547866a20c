"""The library's plan for a benchmark line (no device needed): python tools/describe.py "<line>" level variant"""
import ctypes
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_1704_03092_b200 as stc  # noqa: E402
from paper_1704_03092_b200 import _lib  # noqa: E402
from paper_1704_03092_b200.strassen import Variant, problem_of  # noqa: E402


class _Stub:
    def __init__(self, e):
        st, run = [], 1
        for x in reversed(e):
            st.append(run)
            run *= x
        self.extents, self.strides, self.base_offset, self.data = tuple(e), tuple(reversed(st)), 0, None


def describe(line, level, variant, grid=148):
    spec = stc.parse_benchmark_line(line)
    t = lambda labels: _Stub(spec.tensor_extents(labels))  # noqa: E731
    p = problem_of(spec, t(spec.labels_a), t(spec.labels_b), t(spec.labels_c), level, Variant(variant))
    info = _lib.PlanInfo()
    _lib.check(_lib.lib().stc_plan_describe(ctypes.byref(p), grid, ctypes.byref(info)))
    return info.as_dict()


if __name__ == "__main__":
    print(describe(sys.argv[1], int(sys.argv[2]), sys.argv[3]))
