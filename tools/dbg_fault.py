import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2603_29129_b200 as oz, workloads
for n in (1000, 5000):
    x = workloads.draw("uniform", 3, 1, n); xt = torch.from_numpy(x).cuda()
    os.environ.pop("OZFFT_FAULT_INJECT", None)
    a = oz.Plan(n, 1); ya, ta = a.execute_taps(xt)
    os.environ["OZFFT_FAULT_INJECT"] = "1"
    b = oz.Plan(n, 1); yb, tb = b.execute_taps(xt)
    d = (ya != yb).sum().item()
    print(n, "out diff elems", d, "res diff", (ta["res"] != tb["res"]).sum().item(), "crt diff", (ta["crt"] != tb["crt"]).sum().item(),
          "fwd diff", (a.forward(xt) != b.forward(xt)).sum().item())
