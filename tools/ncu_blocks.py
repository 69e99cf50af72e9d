"""Group an ncu SASS source page into basic blocks by execution count (which
code runs how often): python tools/ncu_blocks.py rep kernel_regex [n]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]; si = h.index("Source"); ii = h.index("Instructions Executed")
seen = set(); seq = []
for r in rows[1:]:
    if len(r) <= max(si, ii) or not r[ii].isdigit():
        continue
    if r[0] in seen:
        continue
    seen.add(r[0])
    seq.append((int(r[ii]), r[si].strip()))
tot = sum(n for n, _ in seq)
print(f"total warp-instr {tot:,}  ({len(seq)} instructions)")
blocks = []; cur = None
for n, src in seq:
    if cur and cur[0] == n:
        cur[1].append(src)
    else:
        cur = [n, [src]]; blocks.append(cur)
agg = {}
for n, srcs in blocks:
    agg.setdefault(n, []).append(srcs)
items = sorted(agg.items(), key=lambda kv: -kv[0] * sum(len(x) for x in kv[1]))
for n, groups in items[:top]:
    cnt = sum(len(x) for x in groups)
    ops = {}
    for g in groups:
        for src in g:
            op = src.split()[0] if not src.startswith("@") else src.split()[1]
            op = op.split(".")[0]
            ops[op] = ops.get(op, 0) + 1
    opstr = ", ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:8])
    print(f"{n:>10,} x {cnt:4d} = {n * cnt / tot * 100:5.1f}%  {opstr}")
