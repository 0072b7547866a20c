"""Per-kernel summary of an ncu report: python tools/ncu_table.py report.ncu-rep"""
import csv
import subprocess
import sys

W = [("gpu__time_duration.sum", "ms"), ("dram__bytes_read.sum", "GB rd"), ("dram__bytes_write.sum", "GB wr"),
     ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM%"),
     ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA%"),
     ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64%"),
     ("lts__t_sector_hit_rate.pct", "L2hit%"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
     ("launch__registers_per_thread", "regs"),
     ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall_lsb")]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
print("| kernel | " + " | ".join(n for _, n in W) + " |")
print("|---|" + "---:|" * len(W))
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")][:60]
    cells = []
    for m, _ in W:
        if m in hdr:
            v = r[hdr.index(m)]
            u = units[hdr.index(m)]
            try:
                f = float(v.replace(",", ""))
                if u in ("byte", "Kbyte", "Mbyte", "Gbyte"):
                    f *= {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}[u]
                elif u in ("nsecond", "usecond", "msecond", "second", "ns", "us", "ms", "s"):
                    f *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3,
                          "ms": 1.0, "s": 1e3}[u]
                cells.append(f"{f:.3f}")
            except ValueError:
                cells.append(v)
        else:
            cells.append("-")
    print(f"| `{name}` | " + " | ".join(cells) + " |")
