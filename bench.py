"""Benchmark of the B200 Strassen tensor-contraction path (one JSON line on rank 0).

Workload (BASELINE.json configs[1], the config the headline metric is quoted on):
  2-level ABC Strassen, float64, permuted non-unit-stride layouts
  C[a,i,b,j] += sum_{e,f} A[e,a,f,b] * B[j,f,i,e], all extents 64 (m = n = k = 4096),
  row-major storage in the label order written, entries uniform[-1, 1] from numpy
  default_rng(seed) (A: seed, B: seed + 1), C = 0.  Synthetic data with the
  benchmark's shapes and distribution (there is no dataset for this path).

A "step" is one contract(spec, A, B, C, level=2, variant=ABC) call.
  value  -- effective GFLOP/s = 2 m n k * steps * ranks / (max over ranks of the
            device time of the timed steps), inputs resident in HBM (384 MiB of
            operands per rank > 126 MB L2, so no explicit L2 flush).
  e2e    -- the same metric through the public API with HOST operands in pinned
            memory: every step uploads A, B, C, contracts and downloads C.
Multi-GPU (torchrun, one process per GPU): the n bundle of an N-times wider
problem is split into N independent shards, one cfg2-sized contraction per rank,
no data-path collective (weak scaling).

--impl reference times the reference algorithm on the host CPU (the C restatement
in oracle/, OpenMP over the jr loop like the reference's thread pool, all host
cores) on a bounded n-shard sample of the same workload.
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

SPEC_LINE = "aibj eafb jfie & a:64;b:64;i:64;j:64;e:64;f:64;"
LEVEL, VARIANT = 2, "abc"
SEED = 2017
# FP64 tensor-core (DMMA) peak of this pool's B200, measured with tools/fp64_peak.cu
# (register-resident mma.sync.m8n8k4/m16n8k4/m16n8k16 f64 loops, 148 SMs, best of 5):
# profiles/fp64_peak_r01.txt.  MEASURED_PEAKS.json has no FP64 entry.
FP64_TC_PEAK_TFLOPS = 37.0
CPU_SAMPLE_J = 8  # --impl reference / cpu_baseline: j extent of the n-shard sample (of 64)


def row_major(ext):
    out, run = [], 1
    for e in reversed(ext):
        out.append(run)
        run *= e
    return tuple(reversed(out))


def make_inputs(spec, rank, j_extent=None):
    """Host arrays (numpy) of A, B, C for this rank's n-shard."""
    import paper_1704_03092_b200 as stc

    ext = dict(spec.extents)
    if j_extent is not None:
        ext["j"] = j_extent
    sp = stc.ContractionSpec(spec.labels_c, spec.labels_a, spec.labels_b, ext)

    def tensor(labels, seed, zero=False):
        e = sp.tensor_extents(labels)
        n = int(np.prod(e))
        data = np.zeros(n) if zero else np.random.default_rng(seed).uniform(-1.0, 1.0, n)
        return stc.DenseTensor(e, row_major(e), data)

    # A is shared by every shard; B and C are the rank's slice of the J bundle
    return sp, tensor(sp.labels_a, SEED), tensor(sp.labels_b, SEED + 1 + 1000 * rank), tensor(sp.labels_c, 0, True)


class ClockSampler:
    """nvidia-smi SM clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.proc = None
        self.idx = device_index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.2)
        return self

    def __exit__(self, *exc):
        self.lines = []
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


def cpu_reference_run(steps: int, warmup: int, j_extent: int):
    """Time the reference algorithm (oracle/ C restatement) on a bounded n-shard."""
    import oracle

    import paper_1704_03092_b200 as stc

    spec = stc.parse_benchmark_line(SPEC_LINE)
    sp, a, b, c = make_inputs(spec, 0, j_extent)
    threads = len(os.sched_getaffinity(0))
    oracle.build()
    times = []
    for i in range(warmup + steps):
        st = oracle.contract(sp, a, b, c, LEVEL, VARIANT, threads=threads)
        if i >= warmup:
            times.append(st["seconds"])
    flops = 2.0 * sp.n_i * sp.n_j * sp.n_p
    value = flops * len(times) / sum(times) / 1e9
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except (OSError, IndexError):
        model = "unknown"
    sample = (f"cfg2 n-shard j={j_extent}/64 (m={sp.n_i}, n={sp.n_j}, k={sp.n_p}), L{LEVEL} {VARIANT.upper()}, "
              f"reference blocking (96,4096,256,8,4,4), {threads} threads, {model}")
    return value, threads, sample, sum(times) / len(times)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    metric = "effective fp64 GFLOPS (2mnk/t) and fraction of FP64 tensor peak, 1/2/4/8 B200"
    config = {"workload": "cfg2: C[a,i,b,j] += A[e,a,f,b] B[j,f,i,e], extents 64 (m=n=k=4096), permuted layouts",
              "level": LEVEL, "variant": VARIANT.upper(), "m": 4096, "n": 4096 * world, "k": 4096,
              "n_per_rank": 4096, "parallelism": f"nsplit{world}" if world > 1 else "single",
              "l2_flush": "none: 384 MiB of operands per rank > 126 MB L2", "seed": SEED}

    if args.impl == "reference":
        if rank != 0:
            return
        value, threads, sample, per_step = cpu_reference_run(args.steps, warmup, CPU_SAMPLE_J)
        line = {"metric": metric, "impl": "reference", "value": value, "unit": "GFLOP/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic uniform[-1,1] (seeded)",
                "config": config,
                "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": threads, "kind": "port",
                                 "sample": sample},
                "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch

    import paper_1704_03092_b200 as stc

    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    spec = stc.parse_benchmark_line(SPEC_LINE)
    sp, a_h, b_h, c_h = make_inputs(spec, rank)
    A, B, C = a_h.to_device(dev), b_h.to_device(dev), c_h.to_device(dev)
    torch.cuda.synchronize()
    flops = 2.0 * sp.n_i * sp.n_j * sp.n_p

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(warmup):
        st = stc.contract(sp, A, B, C, LEVEL, VARIANT, synchronize=False)
    barrier()

    # ---- timed region: K steps, device events, gemm events per step ------------
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
    elapsed = t0.elapsed_time(t1) * 1e-3
    gemm_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    if dist is not None:
        tt = torch.tensor([elapsed], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed = float(tt.item())
    value = flops * args.steps * world / elapsed / 1e9

    # ---- e2e: public API with pinned host operands, H2D + D2H inside each step --
    def pinned(t):
        return stc.DenseTensor(t.extents, t.strides, torch.from_numpy(t.data).pin_memory(), t.base_offset)

    a_p, b_p, c_p = pinned(a_h), pinned(b_h), pinned(c_h)
    for _ in range(2):
        stc.contract(sp, a_p, b_p, c_p, LEVEL, VARIANT)  # warm the staging path
    barrier()
    w0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        stc.contract(sp, a_p, b_p, c_p, LEVEL, VARIANT)
    barrier()
    e2e_elapsed = time.perf_counter() - w0
    if dist is not None:
        tt = torch.tensor([e2e_elapsed], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_elapsed = float(tt.item())
    e2e_value = flops * args.e2e_steps * world / e2e_elapsed / 1e9
    bytes_of = lambda t: t.data.numel() * 8
    h2d = bytes_of(a_p) + bytes_of(b_p) + bytes_of(c_p)
    d2h = bytes_of(c_p)

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (fused DMMA Strassen kernel) ----------
    # achieved = 2mnk / t of the launch (the classical flop count, the
    # metric's own unit; up to (8/7)^L above the pipe's peak in principle).  The flops the
    # tensor pipe actually executes, 7^L leaf products of the padded quadrants, are reported
    # beside it as the pipe utilisation.
    q = 1 << LEVEL  # cfg2's bundles divide by 2^L: no PAD
    alg_flops = flops  # 2 m n k of the contraction one launch performs
    exec_flops = (7 ** LEVEL) * 2.0 * (sp.n_i // q) * (sp.n_j // q) * (sp.n_p // q)
    gemm_avg = sum(gemm_ms) / len(gemm_ms) * 1e-3
    achieved = alg_flops / gemm_avg / 1e12
    traffic = None
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists():
        try:
            traffic = json.loads(tfile.read_text()).get("cfg2_L2_abc_gemm_dram_bytes")
        except (ValueError, OSError):
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": FP64_TC_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_TC_PEAK_TFLOPS, "traffic": traffic,
                "kernel": ("k_strassen_fused (TMA views; A sums by the summing warpgroup, B sums in the DMMA fragment loads)" if st.fast_blocks
                           else "k_strassen_gemm (gather producer, Strassen sums in smem)"),
                "kernel_ms": gemm_avg * 1e3, "kernel_share_of_step": gemm_avg / (elapsed / args.steps),
                "algorithmic_flops_per_launch": alg_flops,
                "algorithmic_unit": "2*m*n*k per contraction (SURVEY.md 8(d))",
                "executed_flops_per_launch": exec_flops,
                "executed_tflops": exec_flops / gemm_avg / 1e12,
                "executed_frac_of_pipe_peak": exec_flops / gemm_avg / 1e12 / FP64_TC_PEAK_TFLOPS,
                "peak_source": "measured FP64 DMMA peak, tools/fp64_peak.cu, burst (MEASURED_PEAKS.json has no FP64)"}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cval, threads, sample, _ = cpu_reference_run(1, 0, CPU_SAMPLE_J)
            cpu = {"value": cval, "unit": "GFLOP/s", "cores": threads, "kind": "port", "sample": sample}
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "port", "sample": f"failed: {exc}"}

    line = {"metric": metric, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": warmup, "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic uniform[-1,1], numpy default_rng(2017/2018)", "config": config,
            "e2e": {"value": e2e_value, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": args.e2e_steps, "timing": "wall clock around contract() on pinned host DenseTensors"},
            "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks.summary(),
            "fraction_of_fp64_peak": value / world / 1e3 / FP64_TC_PEAK_TFLOPS}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
