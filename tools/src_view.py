"""Compact view of an ncu source-page CSV (--print-source sass):
   python tools/src_view.py src.csv [min_exec]   -> idx, exec count, samples, top stalls, SASS."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
minx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot_s = sum(int(r[ix["# Samples"]] or 0) for r in rows[2:])
tot_i = sum(int(r[ix["Instructions Executed"]] or 0) for r in rows[2:])
print(f"total samples {tot_s}  warp-instr {tot_i}")
for k, r in enumerate(rows[2:]):
    ex = int(r[ix["Instructions Executed"]] or 0)
    if ex < minx:
        continue
    s = int(r[ix["# Samples"]] or 0)
    st = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stalls), reverse=True)[:2]
    sts = " ".join(f"{n}={v}" for v, n in st if v)
    print(f"{k:5d} {ex:10d} {s:6d} {sts:32s} {r[ix['Source']].strip()[:70]}")
