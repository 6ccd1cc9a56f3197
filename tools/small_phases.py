"""Per-phase times of k_small_fused (variant build with -DOZ_SMALL_TIMING=1):
    python tools/small_phases.py [n] [reps]   -> per phase: max over CTAs of (stamp - launch start)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_29129_b200 as oz  # noqa: E402
import workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
lib = oz.load_library()
x = torch.from_numpy(workloads.draw("uniform", 0, 1, n)).cuda()
plan = oz.Plan(n, 1)
out = torch.empty_like(x)
names = ["start", "split", "forward", "items", "cl.sync", "finish", "exit"]
acc = []
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if os.environ.get("FLUSH") else None
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
evt = []
for r in range(reps + 3):
    if flush is not None:
        flush.zero_()
    e0.record()
    plan.forward(x, out=out)
    e1.record()
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (64 * 16))()
    assert lib.ozfft_debug_small_times(buf) == 0
    t = np.frombuffer(buf, dtype=np.uint64).reshape(64, 16).astype(np.int64)
    used = t[:, 0] > 0
    t = t[used]
    t0 = t[:, 0].min()
    if r >= 3:
        evt.append(e0.elapsed_time(e1) * 1000.0)
        acc.append([(t[:, k] - t0).max() for k in range(16)])
a = np.median(np.array(acc), axis=0) / 1000.0
print(f"event time per execute {np.median(evt):.2f} us (flush={flush is not None})")
print(f"n={n} Z={os.environ.get('OZFFT_SMALL_Z', '-')} CTAs={used.sum()}  (us from the first CTA's start; median of {reps})")
for k in range(7):
    print(f"  {names[k]:8s} {a[k]:7.2f}")
print(f"  l1 start {a[7]:7.2f}")
extra = ["l0 max", "l0 red", "l1 max", "l1 red", "l2 max", "l2 red", "lK", "sched"]
for k in range(8):
    print(f"  {extra[k]:8s} {a[8 + k]:7.2f}")
