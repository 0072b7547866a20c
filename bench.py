"""Benchmark of the B200 Strassen tensor-contraction path (one JSON line on rank 0).

Headline workload: BASELINE.json configs[4] (cfg5), the config the north star
quotes at 1/2/4/8 GPUs -- 2-level ABC Strassen in FP64,
  C[a,b,c,i,j,k] += sum_{e,f,g} A[a,b,c,e,f,g] * B[e,f,g,i,j,k], all extents 32
  (m = n = k = 32768, 8 GiB per operand), row-major, entries uniform[-1,1) from a
  seed (A: 2017, B: 2018; the counter-based generator stc_fill_uniform, so each
  rank generates exactly its part in HBM), C = 0 before the warm-up.
Synthetic data with the config's shapes and distribution (there is no dataset).

A "step" is one contract(spec, A, B, C, level=2, variant=ABC) call over the
rank's part of the problem.  At N GPUs (torchrun, one process per GPU) the n
bundle is split on its label i (32 / N values per rank, shard.plan_shards):
every rank holds all of A, its slice of B and the full C storage, and contracts
its shard of C -- no data-path collective (strong scaling of one problem).
  value  -- effective GFLOP/s = 2 m n k * steps / (max over ranks of the device
            time of the timed steps): the whole problem's classical flops.
            Operands (24 GiB at N = 1) are far larger than the 126 MB L2: no flush.
  allgather (N > 1) -- the optional NCCL all-gather of the C shards
            (shard.gather_shards), timed separately, and the value with it.
  e2e    -- the same metric through the public API with HOST operands in pinned
            memory: every step uploads the rank's A, B shard and C shard,
            contracts and downloads the C shard (stc_contract_host pipeline).
  secondary (N = 1) -- the north star's bar point (m = n = k = 16384,
            abij-abef-efij, extents 128, L2 ABC) and cfg2 (4096^3 permuted
            layouts, L2 ABC), device-resident; the bar point again with three
            levels (allow_deep), an extra beyond the BASELINE levels.
  roofline -- the fused DMMA kernel's own CUDA events over the timed steps.

--impl reference times the reference's own CPU implementation (strassen_tc,
installed under baseline/_ref; the oracle/ C port when it cannot be imported),
all host cores, on a bounded sample of cfg5: the sub-problem a < 2, i < 2,
e < 4 (m = n = 2048, k = 4096, 34.4 GFLOP: L2 leaves of 512 x 512 x 1024), with
the full tensors' values.  Its rate is reported as measured on that sample (the
reference's own cfg5 n-shard run, tests/golden/big.json, ran at a similar rate:
5.9 GFLOP/s on 8 cores).
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CFG5 = "abcijk abcefg efgijk & a:32;b:32;c:32;i:32;j:32;k:32;e:32;f:32;g:32;"
BAR = "abij abef efij & a:128;b:128;i:128;j:128;e:128;f:128;"
CFG2 = "aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;"
SHARD_LABEL = "i"
LEVEL, VARIANT = 2, "abc"
SEED_A, SEED_B = 2017, 2018
# CPU sample of cfg5: the leading ranges of a, i and e: m = n = 2048, k = 4096
CPU_SAMPLE = {"a": 2, "i": 2, "e": 4}
# FP64 tensor-core (DMMA) peak of this pool's B200, measured with tools/fp64_peak.cu
# (register-resident mma.sync f64 loops, 148 SMs, best of 5): profiles/fp64_peak_r01.txt.
# MEASURED_PEAKS.json has no FP64 entry.
FP64_TC_PEAK_TFLOPS = 37.0
METRIC = "effective fp64 GFLOPS (2mnk/t) and fraction of FP64 tensor peak, 1/2/4/8 B200"


def row_major(ext):
    out, run = [], 1
    for e in reversed(ext):
        out.append(run)
        run *= e
    return tuple(reversed(out))


class ClockSampler:
    """nvidia-smi SM clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.proc = None
        self.idx = device_index
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.2)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except (ValueError, IndexError):
                continue
            for name, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ CPU reference
def _cpu_model():
    try:
        return [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except (OSError, IndexError):
        return "unknown"


def _reference_module():
    """The reference package (baseline/_ref) or None."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "strassen_tc").is_dir():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_stc")
    sys.path.insert(0, str(ref))
    try:
        import strassen_tc  # noqa: F401

        return strassen_tc
    except Exception:  # numba missing or broken: use the port
        sys.path.remove(str(ref))
        return None


def cpu_reference_run(steps: int, warmup: int):
    """Time the reference's CPU path on the bounded cfg5 sample (all host cores).

    The reference itself (strassen_tc.contract from baseline/_ref, kind
    "reference") when importable, else the oracle/ C restatement ("port").  The
    sample's inputs carry the full cfg5 tensors' values (oracle/synth.py)."""
    from oracle import synth

    mod = _reference_module()
    threads = len(os.sched_getaffinity(0))
    if mod is not None:
        spec0 = mod.parse_benchmark_line(CFG5)
        mk, kind = mod.DenseTensor, "reference"
    else:
        import oracle

        import paper_1704_03092_b200 as stc

        oracle.build()
        spec0 = stc.parse_benchmark_line(CFG5)
        mk, kind = stc.DenseTensor, "port"
    full = dict(spec0.extents)
    ext = dict(full)
    ext.update(CPU_SAMPLE)
    sp = type(spec0)(spec0.labels_c, spec0.labels_a, spec0.labels_b, ext)

    def tensor(labels, seed, zero=False):
        e = tuple(ext[x] for x in labels)
        data = np.zeros(int(np.prod(e))) if zero else synth.tensor_values(seed, e, row_major(
            tuple(full[x] for x in labels)), 0)
        return mk(e, row_major(e), data)

    a, b, c = tensor(sp.labels_a, SEED_A), tensor(sp.labels_b, SEED_B), tensor(sp.labels_c, 0, True)
    if mod is not None:
        run = lambda: mod.contract(sp, a, b, c, LEVEL, mod.Variant.ABC, threads=threads).seconds
        # numba compiles on first use: one tiny call outside the measured steps
        tiny = mod.parse_benchmark_line("abij abef efij & a:4;b:4;i:4;j:4;e:4;f:4;")
        ta, tb, tc = (mod.DenseTensor((4,) * 4, row_major((4,) * 4), np.ones(256)) for _ in range(3))
        mod.contract(tiny, ta, tb, tc, LEVEL, mod.Variant.ABC, threads=threads)
    else:
        import oracle

        run = lambda: oracle.contract(sp, a, b, c, LEVEL, VARIANT, threads=threads)["seconds"]
    times = []
    for i in range(warmup + steps):
        t = run()
        if i >= warmup:
            times.append(t)
    flops = 2.0 * sp.n_i * sp.n_j * sp.n_p
    value = flops * len(times) / sum(times) / 1e9
    sample = (f"cfg5 sub-problem " + ", ".join(f"{k}<{v}" for k, v in CPU_SAMPLE.items()) + " "
              f"(m={sp.n_i}, n={sp.n_j}, k={sp.n_p}, {flops / 1e9:.1f} GFLOP per step, full-tensor values), "
              f"L{LEVEL} {VARIANT.upper()}, "
              + ("strassen_tc.contract from baseline/_ref (numba)" if kind == "reference"
                 else "oracle/stc_oracle.c port (OpenMP over jr)")
              + f", {threads} threads, {_cpu_model()}; rate as measured on the sample")
    return value, threads, kind, sample, sum(times) / len(times)


# ------------------------------------------------------------------ GPU arm
def _spec(line):
    import paper_1704_03092_b200 as stc

    return stc.parse_benchmark_line(line)


def _time_config(line, steps, warmup, dev, level=LEVEL):
    """Effective TFLOP/s of ABC at `level` on a device-resident config (secondary keys)."""
    import torch

    import paper_1704_03092_b200 as stc
    from paper_1704_03092_b200.synth import uniform_tensor

    spec = _spec(line)
    a = uniform_tensor(SEED_A, spec.tensor_extents(spec.labels_a), dev)
    b = uniform_tensor(SEED_B, spec.tensor_extents(spec.labels_b), dev)
    ec = spec.tensor_extents(spec.labels_c)
    c = stc.DenseTensor(ec, row_major(ec), torch.zeros(int(np.prod(ec)), dtype=torch.float64, device=dev))
    kw = {"allow_deep": True} if level > 2 else {}
    for _ in range(warmup):
        stc.contract(spec, a, b, c, level, VARIANT, synchronize=False, **kw)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        stc.contract(spec, a, b, c, level, VARIANT, synchronize=False, **kw)
    t1.record(stream)
    torch.cuda.synchronize()
    s = t0.elapsed_time(t1) * 1e-3 / steps
    tf = 2.0 * spec.n_i * spec.n_j * spec.n_p / s / 1e12
    del a, b, c
    torch.cuda.empty_cache()
    return {"line": line, "level": level, "variant": VARIANT.upper(), "ms_per_step": s * 1e3,
            "effective_tflops": tf, "frac_of_fp64_peak": tf / FP64_TC_PEAK_TFLOPS, "steps": steps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    args = ap.parse_args()
    warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    config = {"workload": "cfg5: C[a,b,c,i,j,k] += A[a,b,c,e,f,g] B[e,f,g,i,j,k], extents 32 "
                          "(m=n=k=32768), row-major", "level": LEVEL, "variant": VARIANT.upper(),
              "m": 32768, "n": 32768, "k": 32768, "shard_label": SHARD_LABEL, "n_per_rank": 32768 // world,
              "parallelism": f"nsplit{world}" if world > 1 else "single",
              "l2_flush": "none: 24 GiB of operands at N=1 (A 8 GiB + slices per rank) >> 126 MB L2",
              "seed": [SEED_A, SEED_B], "generator": "counter-based uniform[-1,1) (stc_fill_uniform)"}

    if args.impl == "reference":
        if rank != 0:
            return
        value, threads, kind, sample, per_step = cpu_reference_run(args.steps, warmup)
        line = {"metric": METRIC, "impl": "reference", "value": value, "unit": "GFLOP/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic uniform[-1,1) (seeded, counter-based)", "config": config,
                "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": threads, "kind": kind, "sample": sample},
                "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch

    import paper_1704_03092_b200 as stc
    from paper_1704_03092_b200 import shard
    from paper_1704_03092_b200.synth import uniform_tensor

    dist = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        # STC_BENCH_BACKEND=gloo (a dry run of the multi-rank path on fewer GPUs than ranks:
        # ranks share devices round-robin, the collectives go through host memory)
        backend = os.environ.get("STC_BENCH_BACKEND", "nccl")
        torch.cuda.set_device(local_rank % torch.cuda.device_count())
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    spec = _spec(CFG5)
    ea, eb, ec = (spec.tensor_extents(l) for l in (spec.labels_a, spec.labels_b, spec.labels_c))
    # rank's part: all of A, B[:, shard] (generated as its own compact slice), and the
    # full C storage (the shard is a view; the optional all-gather fills the rest)
    c_full = stc.DenseTensor(ec, row_major(ec), torch.zeros(int(np.prod(ec)), dtype=torch.float64, device=dev))
    sh = shard.plan_shards(spec, c_full, world, SHARD_LABEL)[rank]
    sp = shard.shard_spec(spec, sh)
    A = uniform_tensor(SEED_A, ea, dev)
    ax = spec.labels_b.index(SHARD_LABEL)
    B = uniform_tensor(SEED_B, sp.tensor_extents(sp.labels_b), dev, full_strides=row_major(eb),
                       base=sh.start * row_major(eb)[ax])
    C = shard.shard_tensor(c_full, spec.labels_c, sh)
    A_desc, B_desc, C_desc = A, B, C  # layouts for the plan description (no storage use)
    torch.cuda.synchronize()
    flops_rank = 2.0 * sp.n_i * sp.n_j * sp.n_p
    flops_job = 2.0 * spec.n_i * spec.n_j * spec.n_p

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], device=dev if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(warmup):
        stc.contract(sp, A, B, C, LEVEL, VARIANT, synchronize=False)
    barrier()

    # ---- timed region: K steps, device events; fused-kernel events per step -----
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for e0, e1 in ev:  # torch creates the cudaEvent_t lazily, on first record
        e0.record(stream)
        e1.record(stream)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clocks:
        barrier()
        t0.record(stream)
        launches = 0
        for i in range(args.steps):
            st = stc.contract(sp, A, B, C, LEVEL, VARIANT, kernel_events=ev[i], synchronize=False)
            launches += st.kernel_launches
        t1.record(stream)
        barrier()
    elapsed = max_over_ranks(t0.elapsed_time(t1) * 1e-3)
    gemm_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    value = flops_job * args.steps / elapsed / 1e9

    # ---- optional all-gather of the C shards (NCCL), timed on its own ----------
    allgather = None
    if dist is not None:
        reps = 3
        shard.gather_shards(spec, c_full, rank, world, SHARD_LABEL)  # warm (buffers, NCCL channels)
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(reps):
            shard.gather_shards(spec, c_full, rank, world, SHARD_LABEL)
        g1.record(stream)
        barrier()
        ag = max_over_ranks(g0.elapsed_time(g1) * 1e-3 / reps)
        allgather = {"ms": ag * 1e3, "bytes_per_rank_received": int(np.prod(ec)) * 8 * (world - 1) // world,
                     "value_with_allgather": flops_job / (elapsed / args.steps + ag) / 1e9,
                     "how": "shard.gather_shards: all_gather_into_tensor into a shard-major buffer + one "
                            f"strided copy per shard ({dist.get_backend()})"}
    del c_full
    C = None
    torch.cuda.empty_cache()

    # ---- e2e: public API with pinned host operands, H2D + D2H inside each step --
    def pinned_copy(t):
        h = torch.empty(t.data.numel(), dtype=torch.float64, pin_memory=True)
        h.copy_(t.data)
        return stc.DenseTensor(t.extents, t.strides, h, t.base_offset)

    # Every rank must take the same branch (the timed region holds barriers): the pinned
    # allocations are tried first and the outcome agreed on (min over ranks).
    e2e, err = None, ""
    try:
        a_p, b_p = pinned_copy(A), pinned_copy(B)
        esc = sp.tensor_extents(sp.labels_c)
        c_p = stc.DenseTensor(esc, row_major(esc), torch.zeros(int(np.prod(esc)), dtype=torch.float64,
                                                               pin_memory=True))
    except (RuntimeError, MemoryError) as exc:  # host memory for pinned operands
        err = str(exc)[:200]
    del A, B
    torch.cuda.empty_cache()
    if -max_over_ranks(-float(not err)) > 0:
        stc.contract(sp, a_p, b_p, c_p, LEVEL, VARIANT)  # warm the host pipeline's plans and buffers
        barrier()
        w0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            stc.contract(sp, a_p, b_p, c_p, LEVEL, VARIANT)
        barrier()
        e2e_elapsed = max_over_ranks(time.perf_counter() - w0)
        nbytes = lambda t: t.data.numel() * 8
        e2e = {"value": flops_job * args.e2e_steps / e2e_elapsed / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": nbytes(a_p) + nbytes(b_p) + nbytes(c_p), "d2h_bytes_per_step": nbytes(c_p),
               "steps": args.e2e_steps,
               "timing": "wall clock around contract() on pinned host DenseTensors (per rank: A, B shard, "
                         "C shard), max over ranks"}
    else:
        e2e = {"value": None, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "error": err or "pinned host allocation failed on another rank"}
    a_p = b_p = c_p = None

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (the fused DMMA Strassen kernel) -------
    # achieved = the classical 2 m n k of the launch / its duration
    # (up to (8/7)^L above the pipe's peak in principle); the flops the tensor pipe
    # executes (7^L leaf products of the quadrants) are reported beside it.
    info = stc.describe_plan(sp, A_desc, B_desc, C_desc, LEVEL, VARIANT)
    kernel_name = ("k_strassen_fused on pre-summed operand slots (k_presum), "
                   + ("TMA reduce-add C epilogue" if info["ticketed"] else "dense M + k_accumulate")
                   if info["presum"] else "k_strassen_fused (in-kernel operand sums)")
    q = 1 << LEVEL
    exec_flops = (7 ** LEVEL) * 2.0 * (sp.n_i // q) * (sp.n_j // q) * (sp.n_p // q)
    gemm_avg = sum(gemm_ms) / len(gemm_ms) * 1e-3
    achieved = flops_rank / gemm_avg / 1e12
    traffic = None
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists():
        try:
            traffic = json.loads(tfile.read_text()).get("cfg5_L2_abc_gemm_dram_bytes")
        except (ValueError, OSError):
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": FP64_TC_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_TC_PEAK_TFLOPS, "traffic": traffic,
                "kernel": kernel_name,
                "kernel_ms": gemm_avg * 1e3, "kernel_share_of_step": gemm_avg / (elapsed / args.steps),
                "algorithmic_flops_per_launch": flops_rank,
                "algorithmic_unit": "2*m*n*k of the rank's contraction (SURVEY.md 8(d))",
                "executed_flops_per_launch": exec_flops,
                "executed_tflops": exec_flops / gemm_avg / 1e12,
                "executed_frac_of_pipe_peak": exec_flops / gemm_avg / 1e12 / FP64_TC_PEAK_TFLOPS,
                "peak_source": "builder-measured FP64 DMMA burst peak, tools/fp64_peak.cu (MEASURED_PEAKS.json "
                               "has no FP64 entry)"}

    secondary = None
    if world == 1 and not args.no_secondary:
        secondary = {"bar_16384": _time_config(BAR, 3, 1, dev), "cfg2": _time_config(CFG2, 10, 3, dev),
                     # three levels (allow_deep; beyond the BASELINE levels), the same bar point
                     "bar_16384_level3": _time_config(BAR, 3, 1, dev, level=3)}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cval, threads, kind, sample, _ = cpu_reference_run(1, 0)
            cpu = {"value": cval, "unit": "GFLOP/s", "cores": threads, "kind": kind, "sample": sample}
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "port", "sample": f"failed: {exc}"}

    line = {"metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": warmup, "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic uniform[-1,1) from seeds 2017/2018 (counter-based, generated in HBM)",
            "config": config, "e2e": e2e, "gpu_launches": launches, "roofline": roofline,
            "cpu_baseline": cpu, "clocks": clocks.summary(),
            "fraction_of_fp64_peak": value / world / 1e3 / FP64_TC_PEAK_TFLOPS}
    if allgather is not None:
        line["allgather"] = allgather
    if secondary is not None:
        line["secondary"] = secondary
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
