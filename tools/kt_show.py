"""Summarise tools/kernel_times.sh output: per variant/config, the last execute's kernels."""
import csv
import glob
import sys

for f in sorted(glob.glob("gpurun_out/kt_*.csv")):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    if not rows:
        continue
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    data = [(r[ki].split("(")[0][:34], float(r[vi].replace(",", "")) / 1000) for r in rows[1:]]
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    print(f[len("gpurun_out/kt_"):-4], " ".join("%s=%.1f" % d for d in data[-n:]))
