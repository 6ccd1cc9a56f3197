import sys, torch
sys.path.insert(0, "/root/repo")
import paper_2603_29129_b200 as oz, workloads
for name in ("c1", "c2"):
    cfg = workloads.CONFIGS[name]
    x = torch.from_numpy(workloads.config_input(cfg)).cuda()
    p = oz.Plan(cfg.n, cfg.batch); out = torch.empty_like(x)
    for _ in range(5): p.forward(x, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): p.forward(x, out=out)
    e1.record(); torch.cuda.synchronize()
    print(name, e0.elapsed_time(e1) / 50)
