"""Key metrics per kernel from an ncu report: ncu_summary.py rep [kernel_regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "raw", "--csv"]
if len(sys.argv) > 2:
    args += ["-k", f"regex:{sys.argv[2]}"]
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size"]
stalls = [n for n in h if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    print(r[h.index("Kernel Name")][:70])
    for k in keys:
        if k in h:
            print(f"   {k:70s} {r[h.index(k)]} {rows[1][h.index(k)]}")
    st = sorted(((float(r[h.index(n)] or 0), n) for n in stalls), reverse=True)[:6]
    print("   stalls/issue:", ", ".join(f"{n.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, n in st))
