"""Summarise an ncu source-page CSV: stall reasons and top SASS lines. usage: ncu_stalls.py file.csv [ntop]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {c: sum(float(r[hdr.index(c)] or 0) for r in data) for c in cols}
s = sum(tot.values())
print("stall reasons (% of samples):", ", ".join(f"{c[6:]} {v/s*100:.1f}" for c, v in sorted(tot.items(), key=lambda x: -x[1]) if v / s > 0.005))
i_s, i_src, i_ex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
T = sum(float(r[i_s] or 0) for r in data)
ops = {}
for r in data:
    op = r[i_src].split()[0] if r[i_src].strip() else "?"
    if op.startswith("@"): op = r[i_src].split()[1]
    op = op.split(".")[0]
    ops[op] = ops.get(op, 0) + float(r[i_ex] or 0)
print("executed warp-instructions by opcode:", ", ".join(f"{k} {v:.3g}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:14]))
for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:ntop]:
    top = max(cols, key=lambda c: float(r[hdr.index(c)] or 0))
    print(f"{float(r[i_s])/T*100:5.2f}% {top[6:]:14s} {r[i_src][:80]}")
