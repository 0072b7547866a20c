"""Summarise .ncu-rep captures: python tools/ncu_summary.py rep1 [rep2 ...]  (prints key metrics per kernel)."""
import csv, io, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma_pipe_%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1_%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_%"),
    ("smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct", "stall_long_sb_%"),
    ("smsp__warps_issue_stalled_barrier_per_warp_active.pct", "stall_barrier_%"),
    ("smsp__warps_issue_stalled_math_pipe_throttle_per_warp_active.pct", "stall_math_%"),
    ("smsp__warps_issue_stalled_wait_per_warp_active.pct", "stall_wait_%"),
    ("launch__registers_per_thread", "regs"),
]


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        line = {"kernel": d.get("Kernel Name", "?")[:40]}
        for k, name in KEYS:
            if k in d:
                line[name] = f"{d[k]} {u.get(k, '')}".strip()
        res.append(line)
    return res


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        for line in summarise(rep):
            print(rep.split("/")[-1], " | ".join(f"{k}={v}" for k, v in line.items()))
