"""execute_host (host buffers, copies in the timed region) per sub-batch schedule:
    OZFFT_HOST_SUBS=1,2,4,4,4,1 python tools/e2e_subs.py [config]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_29129_b200 as oz  # noqa: E402
import workloads  # noqa: E402

cfg = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
xh = torch.from_numpy(workloads.config_input(cfg)).pin_memory()
yh = torch.empty_like(xh).pin_memory()
plan = oz.Plan(cfg.n, cfg.batch)
for _ in range(3):
    plan.execute_host(xh, out_host=yh)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.execute_host(xh, out_host=yh)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
t = ts[len(ts) // 2]
gf = cfg.batch * 5 * cfg.n * __import__("math").log2(cfg.n) / (t * 1e-3) / 1e9
print(f"subs={os.environ.get('OZFFT_HOST_SUBS', 'default')}: {t:.3f} ms  {gf:.1f} GFLOP/s e2e")
