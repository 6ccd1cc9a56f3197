"""The paper's accuracy / NTT-count sweep, run on the
GPU path with seeded synthetic inputs and a __float128 reference instead of MPFR:

  inputs  (rand - 0.5) exp(phi randn), phi in {0, 1, 4}  (eq:input-generation)
  n       2^10 .. 2^18
  (K, L)  (inf, 1), (1, 1), (2, 1), (3, 1), (3, 3); K = inf is the
          build's cap K = 8
  counts  total 32-bit NTT + inverse NTT calls per transform, cached omega* NTTs included
          (the paper's Figs. 5/9 count), and the split counts k of x' and omega~* (Fig. 4)
  errors  max componentwise relative error and relative l2 error against the
          __float128 direct DFT (oracle.dft_f128) on all bins (n <= 4096) or 256 seeded bins
  alpha   the four split widths of Fig. 1 (oracle.alpha_formulas)

Writes profiles/<tag>_sweep.json and .md.   python tools/sweep.py [tag] [max_log2n] [dd|ts]
(ts: the paper's triple-single working precision, SURVEY f4 -- the setting of its counts)
(TEST / EVIDENCE tooling: it uses oracle/ only for the float128 reference.)"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_2603_29129_b200 as oz  # noqa: E402
import workloads  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
max_log = int(sys.argv[2]) if len(sys.argv) > 2 else 18
prec = sys.argv[3] if len(sys.argv) > 3 else "dd"
KL = [(8, 1), (1, 1), (2, 1), (3, 1), (3, 3)]
PHIS = [0.0, 1.0, 4.0]
B = 4


def errors(y, x):
    n = x.size
    if n <= 4096:
        bins = np.arange(n)
    else:
        bins = np.sort(np.random.default_rng(n).choice(n, 256, replace=False))
    hi, lo = O.dft_f128(x, bins=bins)
    ref = hi + lo
    d = y[bins] - ref
    with np.errstate(divide="ignore", invalid="ignore"):
        rr = np.abs(d.real / ref.real)
        ri = np.abs(d.imag / ref.imag)
    mx = float(np.nanmax(np.concatenate([rr[np.isfinite(rr)], ri[np.isfinite(ri)]])))
    l2 = float(np.linalg.norm(d) / np.linalg.norm(ref))
    return mx, l2, len(bins)


rows = []
for phi in PHIS:
    for lg in range(10, max_log + 1):
        n = 1 << lg
        x = workloads.phi_input(n, phi, seed=lg * 10 + int(phi), batch=B)
        xt = torch.from_numpy(x).cuda()
        for K, L in KL:
            plan = oz.Plan(n, 1, K=K, L=L, precision=prec)
            per_t, kx = [], []
            for b in range(B):  # one transform at a time: per-transform counts (the paper's max)
                yb = plan.forward(xt[b:b + 1].contiguous()).cpu().numpy()
                st = plan.stats()
                per_t.append(st["fwd_ntts"] + st["inv_ntts"] + st["cached_ntts"])
                kx.append(st["k"][:2])
                if b == 0:
                    y0 = yb[0]
            mx, l2, nb = errors(y0, x[0])
            rows.append({"phi": phi, "n": n, "K": "inf(8)" if K == 8 else K, "L": L, "precision": prec,
                         "alpha": plan.alpha, "k_x": kx[0], "k_x_all": kx, "k_w": st["k"][2:],
                         "ntt_total": max(per_t), "ntt_per_transform": per_t,
                         "ntt_runtime": max(per_t) - st["cached_ntts"],
                         "max_rel_err": mx, "rel_l2_err": l2, "bins": nb})
            print(json.dumps(rows[-1]), flush=True)
            del plan
alpha = {1 << k: O.alpha_formulas(1 << k) for k in range(10, 21)}
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
json.dump({"rows": rows, "alpha_fig1": alpha}, open(os.path.join(ROOT, "profiles", f"{tag}_sweep.json"), "w"),
          indent=1)
md = [f"# Accuracy / NTT-count sweep ({tag}; tools/sweep.py, one B200, precision {prec})", "",
      "Inputs (rand-0.5)exp(phi randn), 4 transforms per point, transform 0 scored against the",
      "__float128 DFT (all bins for n <= 4096, else 256 seeded bins). NTTs = the largest",
      "per-transform count of the 4 (the paper reports maxima), cached omega* NTTs included;",
      "k(Re x', Im x') of transform 0. K = inf is the build's cap K = 8.",
      ("Working precision is double-double (DESIGN ruling 1), so split counts and errors are "
       "not the paper's TS figures; the count laws and the (3,3) / (3,1) totals at phi = 0, 1 are."
       if prec == "dd" else
       "Working precision is the paper's triple-single (SURVEY f4, DESIGN section 15): the "
       "setting of the paper's counts (P:1112, P:1164-1167)."), "",
      "| phi | n | (K, L) | alpha | k(Re x', Im x') | k(Re w, Im w) | NTTs | max rel err | rel l2 err |",
      "|---|---|---|---|---|---|---|---|---|"]
for r in rows:
    md.append(f"| {r['phi']:.0f} | 2^{int(np.log2(r['n']))} | ({r['K']}, {r['L']}) | {r['alpha']} | "
              f"{r['k_x'][0]}, {r['k_x'][1]} | {r['k_w'][0]}, {r['k_w'][1]} | {r['ntt_total']:.0f} | "
              f"{r['max_rel_err']:.2e} | {r['rel_l2_err']:.2e} |")
md += ["", "## Fig. 1: split width alpha in single precision (u = 2^-24; oracle.alpha_formulas)", "",
       "| n | original Ozaki | FFT-based | one-prime NTT | two-prime NTT + CRT |", "|---|---|---|---|---|"]
for n, a in alpha.items():
    md.append(f"| 2^{int(np.log2(n))} | {a['ozaki']} | {a['fft']} | {a['ntt']} | {a['crt']} |")
open(os.path.join(ROOT, "profiles", f"{tag}_sweep.md"), "w").write("\n".join(md) + "\n")
print("wrote", f"profiles/{tag}_sweep.md")
