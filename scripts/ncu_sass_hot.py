"""Dev tool: aggregate ncu source-page stall samples of a kernel by SASS opcode / stall reason.

    python scripts/ncu_sass_hot.py report.ncu-rep [top]
"""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
by_op = defaultdict(lambda: [0, 0])
by_reason = defaultdict(int)
tot = 0
seq = []
for r in rows[1:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    n = int(r[ix["Instructions Executed"]] or 0)
    by_op[op][0] += s
    by_op[op][1] += n
    tot += s
    for c in stall_cols:
        v = int(r[ix[c]] or 0)
        by_reason[c] += v
    seq.append((s, src, {c: int(r[ix[c]] or 0) for c in stall_cols}))
print(f"total samples {tot}")
for op, (s, n) in sorted(by_op.items(), key=lambda x: -x[1][0])[:25]:
    print(f"  {op:10s} samples {s:7d} ({100*s/tot:5.1f}%)  warp-inst {n}")
print("reasons:")
for c, v in sorted(by_reason.items(), key=lambda x: -x[1])[:14]:
    print(f"  {c:24s} {v:7d} ({100*v/tot:5.1f}%)")
print("hottest instructions:")
for s, src, d in sorted(seq, key=lambda x: -x[0])[:top]:
    rs = sorted(d.items(), key=lambda x: -x[1])[:3]
    print(f"  {s:6d}  {src[:60]:60s} " + " ".join(f"{k[6:]}={v}" for k, v in rs if v))
