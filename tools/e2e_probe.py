"""Probe the end-to-end (host-buffer) path: PCIe copy rates and execute_host vs execute."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_29129_b200 as oz  # noqa: E402
import workloads  # noqa: E402

cfg = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
x = torch.from_numpy(workloads.config_input(cfg))
xh = x.pin_memory()
yh = torch.empty_like(xh).pin_memory()
xd = x.cuda()
yd = torch.empty_like(xd)
for name, f in [("H2D", lambda: xd.copy_(xh, non_blocking=True)),
                ("D2H", lambda: yh.copy_(yd, non_blocking=True))]:
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        f()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"{name}: {xh.numel() * 16 / dt / 1e9:.1f} GB/s ({dt * 1e3:.3f} ms for {xh.numel() * 16 >> 20} MiB)")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1):
        xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        yh.copy_(yd, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 10
print(f"H2D || D2H: {dt * 1e3:.3f} ms for both")
plan = oz.Plan(cfg.n, cfg.batch)
for _ in range(3):
    plan.forward(xd, out=yd)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    plan.forward(xd, out=yd)
torch.cuda.synchronize()
print(f"execute (device buffers): {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms")
for _ in range(2):
    plan.execute_host(xh, out_host=yh)
t0 = time.perf_counter()
for _ in range(10):
    plan.execute_host(xh, out_host=yh)
print(f"execute_host: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms")
for B in (1, 2, 4):
    p = oz.Plan(cfg.n, B)
    xs = xd[:B].contiguous()
    ys = torch.empty_like(xs)
    for _ in range(3):
        p.forward(xs, out=ys)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        p.forward(xs, out=ys)
    torch.cuda.synchronize()
    print(f"execute batch {B}: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms "
          f"({(time.perf_counter() - t0) / 10 * 1e3 / B:.3f} per transform)")
