"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container only (it imports the read-only reference checkout):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

The GPU box never runs this and nothing at test time reads /root/reference;
the tests only read the committed .npz/.json outputs.  What is pinned:

* views.npz     -- make_view / quadrant_views scatter + block-scatter vectors
                   (reference scatter.py:26-131, strassen.py:101-127), including
                   the reference's own unit-test goldens (pkg/tests/test_scatter.py).
* terms.json    -- strassen_terms(L) for L = 0..3 (strassen.py:56-94).
* contract.npz  -- small seeded contractions: inputs, reference contract() output
                   for every level x variant, and contract_reference() output
                   (random permuted layouts as in pkg/tests/helpers.py:10-63;
                   float and integer fills; odd extents for PAD).
* cfg1.json     -- BASELINE config 1 (abij-abef-efij, extents 24, row-major,
                   uniform[-1,1] from seed 7 / 8, C = 0): reference L1 ABC output
                   summarised by norms and 4096 sampled entries.
* full.json     -- BASELINE configs 2 and 4 at full size (cfg2: 4096^3 permuted,
                   uniform[-1,1], L1 / L2 ABC; cfg4: 4550 x 3150 x 2970 irregular,
                   normal(0,1), AB and Naive at L1 / L2), row-major, C = 0: the
                   reference's own outputs summarised by norms and 4096 sampled
                   entries (gen_full; run with --full, several minutes on 8 threads).
"""

from __future__ import annotations

import json
import pathlib
import sys

import numpy as np

REF = pathlib.Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

import strassen_tc as st  # noqa: E402
from helpers import permuted_tensor, random_spec  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent


def row_major_strides(extents):
    s, step = [], 1
    for e in reversed(extents):
        s.append(step)
        step *= e
    return tuple(reversed(s))


def gen_views():
    cases = []
    # the reference unit-test goldens (pkg/tests/test_scatter.py:17-29,32-38,73-77)
    cases.append(dict(ext=(8, 2, 4), strides=(1, 8, 16), base=0, rows="ac", cols="d",
                      labels="dca", rb=8, cb=4, level=0))
    cases.append(dict(ext=(16, 8), strides=(1, 16), base=0, rows="a", cols="b", labels="ab", rb=8, cb=4, level=0))
    cases.append(dict(ext=(7, 7), strides=(1, 7), base=0, rows="a", cols="b", labels="ab", rb=4, cb=4, level=1))
    cases.append(dict(ext=(3, 3), strides=(1, 3), base=2, rows="a", cols="b", labels="ab", rb=2, cb=2, level=0))
    # BASELINE config shapes, small extents, several levels
    cases.append(dict(ext=(6, 4, 5, 2), strides=row_major_strides((6, 4, 5, 2)), base=0, rows="ab", cols="ef",
                      labels="eafb", rb=8, cb=4, level=2))
    cases.append(dict(ext=(5, 7, 3, 6, 2), strides=row_major_strides((5, 7, 3, 6, 2)), base=3, rows="abc",
                      cols="ef", labels="eafbc", rb=8, cb=4, level=1))
    rng = np.random.default_rng(99)
    for _ in range(40):
        ndim = int(rng.integers(2, 5))
        ext = tuple(int(rng.integers(1, 7)) for _ in range(ndim))
        nrow = int(rng.integers(1, ndim))
        labels = "pqrstu"[:ndim]
        t = permuted_tensor(ext, int(rng.integers(2**31)))
        cases.append(dict(ext=ext, strides=t.strides, base=int(rng.integers(0, 5)), rows=labels[:nrow],
                          cols=labels[nrow:], labels=labels, rb=int(rng.choice([2, 4, 8])),
                          cb=int(rng.choice([2, 4])), level=int(rng.integers(0, 3))))
    arrays = {}
    meta = []
    for k, cs in enumerate(cases):
        n = int(np.prod(cs["ext"]))
        span = cs["base"] + sum((e - 1) * s for e, s in zip(cs["ext"], cs["strides"])) + 1
        t = st.DenseTensor(cs["ext"], cs["strides"], np.zeros(max(span, n)), cs["base"])
        axes = {lab: i for i, lab in enumerate(cs["labels"])}
        v = st.make_view(t, cs["rows"], cs["cols"], axes, cs["rb"], cs["cb"])
        views = {0: v} if cs["level"] == 0 else st.quadrant_views(v, cs["level"])
        for q, qv in views.items():
            arrays[f"c{k}_q{q}_rscat"] = qv.rscat
            arrays[f"c{k}_q{q}_cscat"] = qv.cscat
            arrays[f"c{k}_q{q}_rbs"] = qv.rbs
            arrays[f"c{k}_q{q}_cbs"] = qv.cbs
        meta.append(dict(cs, ext=list(cs["ext"]), strides=list(cs["strides"]), nquads=len(views)))
    np.savez_compressed(OUT / "views.npz", **arrays)
    (OUT / "views.json").write_text(json.dumps(meta, indent=1))


def gen_terms():
    out = {}
    for level in range(4):
        out[str(level)] = [[list(map(list, t.a_ops)), list(map(list, t.b_ops)), list(map(list, t.c_ops))]
                           for t in st.strassen_terms(level, allow_deep=True)]
    (OUT / "terms.json").write_text(json.dumps(out))


def gen_contract():
    rng = np.random.default_rng(31337)
    specs = []
    for _ in range(16):
        specs.append((random_spec(rng, max_labels=3, max_extent=24, max_size=36), "random"))
    for _ in range(4):
        specs.append((random_spec(rng, max_labels=3, max_extent=24, max_size=36), "int"))
    for line in ("ab ac cb & a:7;b:13;c:7;", "abc dca db & a:7;b:13;c:3;d:13;",
                 "abcd aebf dfce & a:3;b:4;c:2;d:5;e:4;f:3;", "ab ac cb & a:24;b:20;c:16;"):
        specs.append((st.parse_benchmark_line(line), "random"))
    specs.append((st.parse_benchmark_line("ab ac cb & a:24;b:20;c:16;"), "int"))
    arrays, meta = {}, []
    for k, (spec, fill) in enumerate(specs):
        seed = int(rng.integers(2**31))
        kw = dict(fill="int", int_bound=1024) if fill == "int" else {}
        a = permuted_tensor(spec.tensor_extents(spec.labels_a), seed, **kw)
        b = permuted_tensor(spec.tensor_extents(spec.labels_b), seed + 1, **kw)
        c = permuted_tensor(spec.tensor_extents(spec.labels_c), seed + 2, **kw)
        for name, t in (("a", a), ("b", b), ("c0", c)):
            arrays[f"k{k}_{name}"] = t.data
        cref = c.copy()
        st.contract_reference(spec, a, b, cref)
        arrays[f"k{k}_classical"] = cref.data
        runs = []
        for level in (0, 1, 2):
            for variant in st.Variant:
                cc = c.copy()
                s = st.contract(spec, a, b, cc, level, variant)
                arrays[f"k{k}_L{level}_{variant.value}"] = cc.data
                runs.append(dict(level=level, variant=variant.value, leaf=s.leaf_multiplies,
                                 total_flops=s.total_flops, fast_blocks=s.fast_blocks, slow_blocks=s.slow_blocks,
                                 fast_updates=s.fast_updates, slow_updates=s.slow_updates,
                                 rel_err=st.relative_error(cc, cref)))
        meta.append(dict(line=st.to_benchmark_line(spec), labels=[spec.labels_c, spec.labels_a, spec.labels_b],
                         fill=fill, seed=seed, strides=dict(a=list(a.strides), b=list(b.strides),
                                                             c=list(c.strides)), runs=runs))
    np.savez_compressed(OUT / "contract.npz", **arrays)
    (OUT / "contract.json").write_text(json.dumps(meta, indent=1))


def gen_cfg1():
    spec = st.parse_benchmark_line("abij abef efij & a:24;b:24;i:24;j:24;e:24;f:24;")
    ext = (24, 24, 24, 24)
    rs = row_major_strides(ext)
    a = st.DenseTensor(ext, rs, np.random.default_rng(7).uniform(-1.0, 1.0, 24**4))
    b = st.DenseTensor(ext, rs, np.random.default_rng(8).uniform(-1.0, 1.0, 24**4))
    c = st.DenseTensor(ext, rs, np.zeros(24**4))
    s = st.contract(spec, a, b, c, 1, st.Variant.ABC)
    idx = np.random.default_rng(11).choice(24**4, 4096, replace=False)
    out = dict(line=st.to_benchmark_line(spec), seed_a=7, seed_b=8, level=1, variant="abc",
               leaf_multiplies=s.leaf_multiplies, total_flops=s.total_flops,
               frob=float(np.sqrt(np.sum(c.data**2))), sum=float(np.sum(c.data)),
               sample_index=idx.tolist(), sample_value=c.data[idx].tolist())
    (OUT / "cfg1.json").write_text(json.dumps(out))


FULL = [
    # (name, line, fill, seeds (A, B), runs)
    ("cfg2", "aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;", "uniform", (2017, 2018),
     [(1, "abc"), (2, "abc")]),
    ("cfg4", "abcij eafbc ifje & a:50;b:7;c:13;i:70;j:45;e:90;f:33;", "normal", (4, 5),
     [(1, "ab"), (2, "ab"), (1, "naive"), (2, "naive")]),
]


def gen_full():
    out = []
    for name, line, fill, (sa, sb), runs in FULL:
        spec = st.parse_benchmark_line(line)

        def tensor(labels, seed):
            ext = tuple(spec.extents[x] for x in labels)
            n = int(np.prod(ext))
            rng = np.random.default_rng(seed)
            data = rng.uniform(-1.0, 1.0, n) if fill == "uniform" else rng.standard_normal(n)
            return st.DenseTensor(ext, row_major_strides(ext), data)

        a, b = tensor(spec.labels_a, sa), tensor(spec.labels_b, sb)
        ext_c = tuple(spec.extents[x] for x in spec.labels_c)
        nc = int(np.prod(ext_c))
        idx = np.random.default_rng(12).choice(nc, 4096, replace=False)
        for level, variant in runs:
            c = st.DenseTensor(ext_c, row_major_strides(ext_c), np.zeros(nc))
            s = st.contract(spec, a, b, c, level, st.Variant(variant), threads=8)
            out.append(dict(name=name, line=line, fill=fill, seed_a=sa, seed_b=sb, level=level, variant=variant,
                            seconds=s.seconds, leaf_multiplies=s.leaf_multiplies,
                            frob=float(np.sqrt(np.sum(c.data ** 2))), sum=float(np.sum(c.data)),
                            sample_index=idx.tolist(), sample_value=c.data[idx].tolist()))
            print(name, level, variant, f"{s.seconds:.1f} s", flush=True)
    (OUT / "full.json").write_text(json.dumps(out))


if __name__ == "__main__":
    if "--full" in sys.argv:
        gen_full()
    else:
        gen_views()
        gen_terms()
        gen_contract()
        gen_cfg1()
    print("golden fixtures written to", OUT)
