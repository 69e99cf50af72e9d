"""Summarise an ncu source page (SASS): instructions executed and stall
samples grouped by opcode, top SASS lines. Usage: ncu_hot.py rep kernel_regex"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
si, ii, ti = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ops_i, ops_s = Counter(), Counter()
tot_i = tot_s = 0
top = []
for r in rows[1:]:
    if len(r) <= max(ti, ii, si) or not r[ii].isdigit():
        continue
    op = r[si].strip().split()[0] if r[si].strip() else "?"
    if op.startswith("@"):
        op = r[si].strip().split()[1]
    op = op.split(".")[0]
    n, s = int(r[ii]), int(r[ti] or 0)
    ops_i[op] += n
    ops_s[op] += s
    tot_i += n
    tot_s += s
    top.append((s, n, r[si].strip()[:90]))
print(f"warp-instructions {tot_i:,}  stall samples {tot_s:,}")
for op, n in ops_i.most_common(25):
    print(f"  {op:10s} inst {n / tot_i * 100:5.1f}%  stall {ops_s[op] / max(tot_s, 1) * 100:5.1f}%")
print("top stall lines:")
for s, n, src in sorted(top, reverse=True)[:25]:
    print(f"  {s:7d} {n:10d}  {src}")
