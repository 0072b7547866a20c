"""Reference outputs for the BASELINE configs that are too large to pin whole:
cfg3 (the shape sweep, both readings) and cfg5 (the multi-GPU config).

Run in the build container only (it imports the read-only reference checkout):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_big_golden.py [--only NAME]

Inputs come from the counter-based generator of oracle/synth.py (uniform[-1,1)
from a seed, value = f(seed, flat index in the full tensor)), so the GPU tests
regenerate the same bits on the device with stc_fill_uniform.  For every case
the reference's own ``contract`` (strassen.py:141-207, ABC at the config's
level, 8 threads) runs on the full problem when that is affordable on this CPU
(cfg3 in the 2^24 reading: 137 GFLOP) and otherwise on one n-shard: the J
label ``i`` restricted to [0, stop) -- a slice of B and C with the full
tensors' strides and values (SURVEY.md section 8(c), cfg3 literal and cfg5
rows).  The output (C starts at 0) is summarised by its Frobenius norm, its sum
and 4096 sampled entries (indices into the compact row-major shard of C); the
GPU tests compare both the GPU result restricted to that shard and a GPU run on
the shard itself.  Writes tests/golden/big.json.
"""

from __future__ import annotations

import json
import pathlib
import sys
import time

import numpy as np

REF = pathlib.Path("/root/reference/pkg")
ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(ROOT))

import strassen_tc as st  # noqa: E402

from oracle import synth  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent / "big.json"
SEED_A, SEED_B = 2017, 2018


def cases():
    out = []
    for na in (16, 32, 64, 128, 256):
        ni = 16384 // na  # literal reading: m * n = 2^28, 2.2 TFLOP -> one 1/16 n-shard
        out.append(dict(name=f"cfg3-literal-Na{na}", line=f"abij abef efij & a:{na};b:{na};i:{ni};j:{ni};e:64;f:64;",
                        shard_label="i", shard_stop=ni // 16, levels=[1, 2]))
    for na in (16, 32, 64, 128, 256):
        ni = 4096 // na  # 2^24 reading: 137 GFLOP -> the whole problem
        out.append(dict(name=f"cfg3-2p24-Na{na}", line=f"abij abef efij & a:{na};b:{na};i:{ni};j:{ni};e:64;f:64;",
                        shard_label="i", shard_stop=ni, levels=[1, 2]))
    out.append(dict(name="cfg5", line="abcijk abcefg efgijk & a:32;b:32;c:32;i:32;j:32;k:32;e:32;f:32;g:32;",
                    shard_label="i", shard_stop=1, levels=[2]))
    return out


def row_major(ext):
    s, run = [], 1
    for e in reversed(ext):
        s.append(run)
        run *= e
    return tuple(reversed(s))


def run_case(cs, threads=8):
    spec = st.parse_benchmark_line(cs["line"])
    lab, stop = cs["shard_label"], cs["shard_stop"]
    full = {l: spec.extents[l] for l in spec.extents}
    shard_ext = dict(full)
    shard_ext[lab] = stop
    sp = st.ContractionSpec(spec.labels_c, spec.labels_a, spec.labels_b, shard_ext)

    def shard_tensor(labels, seed):
        e_full = tuple(full[x] for x in labels)
        e = tuple(shard_ext[x] for x in labels)
        data = synth.tensor_values(seed, e, row_major(e_full), 0)  # slice [0, stop) of `lab`: base 0
        return st.DenseTensor(e, row_major(e), data)

    t0 = time.time()
    a = shard_tensor(spec.labels_a, SEED_A)
    b = shard_tensor(spec.labels_b, SEED_B)
    ext_c = tuple(shard_ext[x] for x in spec.labels_c)
    nc = int(np.prod(ext_c))
    idx = np.sort(np.random.default_rng(12).choice(nc, 4096, replace=False))
    print(cs["name"], f"inputs {time.time() - t0:.1f} s", flush=True)
    res = []
    for level in cs["levels"]:
        c = st.DenseTensor(ext_c, row_major(ext_c), np.zeros(nc))
        s = st.contract(sp, a, b, c, level, st.Variant.ABC, threads=threads)
        res.append(dict(cs, level=level, variant="abc", seed_a=SEED_A, seed_b=SEED_B, generator="oracle/synth.py",
                        shard_line=st.to_benchmark_line(sp), seconds=s.seconds, threads=threads,
                        leaf_multiplies=s.leaf_multiplies, frob=float(np.sqrt(np.sum(c.data ** 2))),
                        sum=float(np.sum(c.data)), sample_index=idx.tolist(), sample_value=c.data[idx].tolist()))
        print(cs["name"], "L", level, f"{s.seconds:.1f} s", f"{s.effective_gflops:.2f} GF/s", flush=True)
    return res


def main():
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    done = json.loads(OUT.read_text()) if OUT.exists() else []
    have = {(d["name"], d["level"]) for d in done}
    for cs in cases():
        if only and not cs["name"].startswith(only):
            continue
        if all((cs["name"], l) in have for l in cs["levels"]):
            continue
        done = [d for d in done if d["name"] != cs["name"]] + run_case(cs)
        OUT.write_text(json.dumps(done))  # after every case: the run is resumable
    print("wrote", OUT)


if __name__ == "__main__":
    main()
