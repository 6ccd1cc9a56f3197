"""Summarise an ncu source page (--page source --csv --print-source sass): stall samples by
opcode class and the hottest instructions.   python tools/sass_hot.py file.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
stall_cols = [k for k in hdr if k.startswith("stall_") or "Stall" in k]
tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
ops = defaultdict(lambda: [0.0, 0])
for r in data:
    op = r[ix["Source"]].strip().split()[0] if r[ix["Source"]].strip() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].strip().split()[1]
    op = op.split(".")[0]
    ops[op][0] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ops[op][1] += int(float(r[ix["Instructions Executed"]] or 0))
ninst = sum(v[1] for v in ops.values())
print(f"total samples {tot:.0f}, warp-instructions {ninst}")
for op, (s, n) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:20]:
    print(f"  {op:10s} samples {s / tot:6.3f}  inst {n / ninst:6.3f}")
print("hottest:")
for r in sorted(data, key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:top]:
    print(f"  {float(r[ix['Warp Stall Sampling (All Samples)']]) / tot:6.3f} {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:70]}")
sc = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
print("stall totals:")
tots = {k: sum(float(r[ix[k]] or 0) for r in data) for k in sc}
for k, v in sorted(tots.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {k:22s} {v / tot:6.3f}")
print("hottest with reasons:")
for r in sorted(data, key=lambda r: -float(r[ix['Warp Stall Sampling (All Samples)']] or 0))[:12]:
    rs = sorted(((float(r[ix[k]] or 0), k) for k in sc), reverse=True)[:3]
    print(f"  {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:48]:48s} " + " ".join(f"{k[6:]}={v:.0f}" for v, k in rs))
