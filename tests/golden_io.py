"""Loaders for the committed golden fixtures (tests/golden/, made by make_golden.py
from the reference itself)."""

import json
import pathlib

import numpy as np

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"


def contract_cases():
    meta = json.loads((GOLDEN / "contract.json").read_text())
    arrays = np.load(GOLDEN / "contract.npz")
    return meta, arrays


def view_cases():
    meta = json.loads((GOLDEN / "views.json").read_text())
    arrays = np.load(GOLDEN / "views.npz")
    return meta, arrays


def terms():
    return json.loads((GOLDEN / "terms.json").read_text())


def cfg1():
    return json.loads((GOLDEN / "cfg1.json").read_text())


def case_operands(DenseTensor, meta, arrays, k):
    """(A, B, C0) DenseTensors of golden contract case k (host storage)."""
    m = meta[k]
    st = m["strides"]
    from_line = m["line"]
    return (DenseTensor(_extents(m, "a"), st["a"], arrays[f"k{k}_a"].copy()),
            DenseTensor(_extents(m, "b"), st["b"], arrays[f"k{k}_b"].copy()),
            DenseTensor(_extents(m, "c"), st["c"], arrays[f"k{k}_c0"].copy()))


def _extents(m, which):
    labels_c, labels_a, labels_b = m["labels"]
    ext = dict(item.split(":") for item in m["line"].split("&")[1].strip().strip(";").split(";"))
    labels = {"a": labels_a, "b": labels_b, "c": labels_c}[which]
    return tuple(int(ext[l]) for l in labels)
