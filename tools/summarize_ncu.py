"""Summarise ncu evidence into profiles/ (run here, on the CPU box, after gpurun).
    python tools/summarize_ncu.py <evidence dir> <round tag>"""
import csv
import json
import os
import subprocess
import sys

ev, tag = sys.argv[1], sys.argv[2]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
prof = os.path.join(root, "profiles")
os.makedirs(prof, exist_ok=True)

# ---- launch list -> per-kernel time share + DRAM traffic per launch
rows = list(csv.reader(open(os.path.join(ev, "launches_c3.csv"))))
hdr, agg, order = None, {}, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].split("(")[0].replace("void ", "")
        if k not in agg:
            order.append(k)
        a = agg.setdefault(k, {})
        a[d["Metric Name"]] = a.get(d["Metric Name"], 0.0) + float(d["Metric Value"].replace(",", ""))
        a.setdefault("_ids", set()).add(d["ID"])
tot = sum(v.get("gpu__time_duration.sum", 0) for v in agg.values())
stage_of = {"k_split_max": "split_max", "k_split_digits": "split_digits", "k_col_fwd": "col_fwd",
            "k_row_fused": "row_fused", "k_col_inv_crt": "col_inv", "k_col_inv": "col_inv",
            "k_finish_dd": "crt_finish", "k_crt_finish": "crt_finish"}
traffic = {}
lines = [f"# ncu launch list, c3 forward execute ({tag}); cold-cache, serialised: compare shares\n",
         "| kernel | launches | time (us) | share | DRAM read (MB) | DRAM write (MB) |",
         "|---|---|---|---|---|---|"]
for k in order:
    v = agg[k]
    nl = len(v["_ids"])
    t = v.get("gpu__time_duration.sum", 0)
    rd, wr = v.get("dram__bytes_read.sum", 0), v.get("dram__bytes_write.sum", 0)
    lines.append(f"| {k} | {nl} | {t / 1e3:.1f} | {t / tot:.3f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} |")
    base = k.split("<")[0]
    if base in stage_of:
        traffic[stage_of[base]] = (rd + wr) / nl  # per launch
open(os.path.join(prof, f"{tag}_launches_c3.md"), "w").write("\n".join(lines) + "\n")
tf = os.path.join(prof, "ncu_traffic.json")
allt = json.load(open(tf)) if os.path.exists(tf) else {}
allt["c3"] = traffic
allt["_about"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes) from the ncu "
                  f"launch list of tools/profile_step.py c3 ({tag}); read by bench.py 'traffic'")
json.dump(allt, open(tf, "w"), indent=1)

# ---- full captures -> key metrics
want = ["Duration", "Compute (SM) Throughput", "DRAM Throughput", "Memory Throughput",
        "Issue Slots Busy", "Executed Ipc Active", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "L1/TEX Hit Rate", "L2 Hit Rate", "SM Frequency"]
raw_keys = ["sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "smsp__inst_executed.sum",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed.avg.per_cycle_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active"]
def pages(f):
    """(details, raw, source CSV path) of a capture: an .ncu-rep, or its CSV pages exported on
    the box by tools/ncu_full_csv.sh (<name>_details.csv, _raw.csv, _sass.csv)."""
    if f.endswith(".ncu-rep"):
        rep = os.path.join(ev, f)
        det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        name = f.replace(".ncu-rep", "")
        src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        tmp = os.path.join(ev, name + "_sass.csv")
        open(tmp, "w").write(src)
        return name, det, raw, tmp
    name = f[:-len("_details.csv")]
    return (name, open(os.path.join(ev, f)).read(), open(os.path.join(ev, name + "_raw.csv")).read(),
            os.path.join(ev, name + "_sass.csv"))


for f in sorted(os.listdir(ev)):
    if not (f.endswith(".ncu-rep") or f.endswith("_details.csv")):
        continue
    name, det, raw, tmp = pages(f)
    out = [f"# {name} ({tag})", ""]
    r = list(csv.reader(det.splitlines()))
    h = r[0]
    for row in r[1:]:
        d = dict(zip(h, row))
        if d.get("Metric Name") in want:
            out.append(f"{d['Metric Name']:45s} {d['Metric Value']} {d['Metric Unit']}")
    rr = list(csv.reader(raw.splitlines()))
    d = dict(zip(rr[0], rr[2])) if len(rr) > 2 else {}
    stalls = []
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                stalls.append((int(v.replace(",", "")), k[33:]))
            except ValueError:
                pass
    out.append("")
    for k in raw_keys:
        out.append(f"{k:70s} {d.get(k)}")
    s = sum(x for x, _ in stalls) or 1
    out.append("\nwarp stall samples (share):")
    for x, k in sorted(stalls, reverse=True)[:10]:
        out.append(f"  {x / s:6.3f} {k}")
    hot = subprocess.run([sys.executable, os.path.join(root, "tools", "sass_hot.py"), tmp, "15"],
                         capture_output=True, text=True).stdout
    out.append("\nSASS opcode mix and hottest instructions (tools/sass_hot.py):")
    out.append(hot)
    open(os.path.join(prof, f"{tag}_{name}.txt"), "w").write("\n".join(out) + "\n")
print(open(os.path.join(prof, f"{tag}_launches_c3.md")).read())
