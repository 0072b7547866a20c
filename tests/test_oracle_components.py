"""CPU: the oracle's component calls (pack_a / pack_b / microkernel restated in
oracle/stc_oracle.c) pinned bitwise to the REFERENCE's outputs
(tests/golden/components.npz, made by tests/golden/make_components_golden.py running
kernels.py:166-233 of the reference)."""

import json
import pathlib

import numpy as np

import oracle

GOLD = pathlib.Path(__file__).resolve().parent / "golden"


def load():
    return json.loads((GOLD / "components.json").read_text()), np.load(GOLD / "components.npz")


def test_oracle_pack_panels_match_reference_bitwise():
    meta, arr = load()
    assert len(meta["pack"]) >= 14
    for k, cs in enumerate(meta["pack"]):
        key = f"pack{k}"
        rows = [arr[f"{key}_r{t}"] for t in range(cs["nviews"])]
        cols = [arr[f"{key}_c{t}"] for t in range(cs["nviews"])]
        want = arr[key + "_out"]
        out, fast, slow = oracle.pack_panel(cs["which"], arr[key + "_data"], rows, cols, cs["rb"], cs["cb"], cs["coeffs"],
                                            cs["x"], cs["k"], depth=want.shape[1], row_unit=cs["row_unit"],
                                            col_unit=cs["col_unit"], force_slow=cs["force_slow"])
        kc = cs["k"][1] - cs["k"][0]
        assert out.shape == want.shape, (k, out.shape, want.shape)
        assert np.array_equal(out[:, :kc].view(np.int64), want[:, :kc].view(np.int64)), k
        assert (fast, slow) == (cs["fast"], cs["slow"]), k


def test_oracle_microkernel_matches_reference_bitwise():
    meta, arr = load()
    for k, cs in enumerate(meta["micro"]):
        key = f"micro{k}"
        c = arr[key + "_before"].copy()
        tg = [(arr[f"{key}_r{g}"], arr[f"{key}_c{g}"], i0, j0, co, cs["row_unit"], cs["col_unit"])
              for g, (i0, j0, co) in enumerate(cs["targets"])]
        fast, slow = oracle.microkernel(arr[key + "_a"], arr[key + "_b"], cs["k"], c, tg, force_slow=cs["force_slow"])
        assert np.array_equal(c.view(np.int64), arr[key + "_after"].view(np.int64)), k
        assert (fast, slow) == (cs["fast"], cs["slow"]), k
