"""Per-CUDA-source-line instruction counts and stall samples from an ncu
report (source page, cuda,sass view). Usage: ncu_lines.py rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
inst = defaultdict(int)
stall = defaultdict(int)
src = {}
fname = None
rows = csv.reader(io.StringIO(out))
hdr = None
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0].isdigit():  # a CUDA line row
        cur = (fname, int(r[0]))
        src[cur] = r[1][:80]
        try:
            inst[cur] += int(r[hdr.index("Instructions Executed")] or 0)
            stall[cur] += int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            pass
tot = sum(inst.values()) or 1
ts = sum(stall.values()) or 1
print(f"total warp-instructions {tot:,}")
for k in sorted(inst, key=lambda k: -inst[k])[:top]:
    print(f"{inst[k] / tot * 100:5.1f}% inst {stall[k] / ts * 100:5.1f}% stall  {k[0]}:{k[1]}  {src[k]}")
