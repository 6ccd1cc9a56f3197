"""Run W warm-up executes + 1 execute of a config's forward pass (for ncu captures).
    python tools/profile_step.py [config] [warmup]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_29129_b200 as oz  # noqa: E402
import workloads  # noqa: E402

cfg = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 2
x = torch.from_numpy(workloads.config_input(cfg)).cuda()
plan = oz.Plan(cfg.n, cfg.batch)
out = torch.empty_like(x)
for _ in range(warm + 1):
    plan.forward(x, out=out)
torch.cuda.synchronize()
print("ok", cfg.name, plan.m, oz.kernel_launches())
