"""Row-kernel item split (OZFFT_ROW_Z) at small batches: ms per execute of c3-size transforms
for batch B:  OZFFT_ROW_Z=z python tools/row_z.py B [B ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_29129_b200 as oz  # noqa: E402
import workloads  # noqa: E402

n = 1 << 18
for B in [int(a) for a in sys.argv[1:]]:
    x = torch.from_numpy(workloads.draw("uniform", 2, B, n)).cuda()
    plan = oz.Plan(n, B)
    out = torch.empty_like(x)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        plan.forward(x, out=out)
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.forward(x, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"Z={os.environ.get('OZFFT_ROW_Z', '-')} B={B}: {ts[len(ts) // 2] * 1000:.1f} us "
          f"({ts[len(ts) // 2] * 1000 / B:.1f} per transform)")
