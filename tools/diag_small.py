import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import oracle
import paper_1704_03092_b200 as stc
def rm(ext):
    out, run = [], 1
    for e in reversed(ext): out.append(run); run *= e
    return tuple(reversed(out))
lines = sys.argv[1:] or ["ab ac cb & a:128;b:128;c:64;", "ab ca cb & a:128;b:128;c:64;", "ab ac cb & a:128;b:128;c:16;",
                         "ab ca cb & a:128;b:128;c:16;", "ab ca cb & a:128;b:128;c:32;", "ab ca cb & a:256;b:128;c:16;"]
for line in lines:
    spec = stc.parse_benchmark_line(line)
    def T(labels, seed):
        ext = spec.tensor_extents(labels)
        return stc.DenseTensor(ext, rm(ext), np.random.default_rng(seed).uniform(-1, 1, int(np.prod(ext))))
    a, b = T(spec.labels_a, 7), T(spec.labels_b, 8)
    c0 = stc.DenseTensor(spec.tensor_extents(spec.labels_c), rm(spec.tensor_extents(spec.labels_c)), np.zeros(spec.n_i * spec.n_j))
    ref = c0.copy(); oracle.contract_reference(spec, a, b, ref, threads=8)
    for kw in ({}, {"force_slow": True}):
        c = c0.copy()
        stc.contract(spec, a, b, c, 0, "abc", **kw)
        err = oracle.relative_error(c, ref)
        bad = np.argwhere(np.abs(c.data - ref.data) > 1e-9 * (1 + np.abs(ref.data))).ravel()
        print(line, kw, f"{err:.3e}", "bad", bad.size, bad[:8], flush=True)
if len(sys.argv) > 1 and sys.argv[1].startswith("abij"):
    # decode the bad elements of the last run into (I row, J col) of the matricised C
    bad_rows = sorted(set(((bad // 576) % 24 * 1 + (bad // 13824) * 0).tolist()))
    aa, bb = bad // 13824, (bad // 576) % 24
    ii, jj = (bad // 24) % 24, bad % 24
    rowI = aa + 24 * bb      # reference linearisation, first label fastest
    colJ = ii + 24 * jj
    print("I rows", sorted(set(rowI.tolist()))[:10], "... count", len(set(rowI.tolist())), "min/max", rowI.min(), rowI.max())
    print("J cols", sorted(set(colJ.tolist()))[:10], "... count", len(set(colJ.tolist())), "min/max", colJ.min(), colJ.max())
    d = (c.data - ref.data)[bad]
    print("diff sample", d[:6], "ref sample", ref.data[bad][:6])
