"""Stage breakdown of the single-transform shard path at N = 1 vs the batched execute of the
same transform (c3 row 0):  python tools/single_prof.py [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_29129_b200 as oz  # noqa: E402
import workloads  # noqa: E402

cfg = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n = cfg.n
x = torch.from_numpy(workloads.draw(cfg.dist, cfg.seed, cfg.batch, n, rows=slice(0, 1))).cuda()
plan = oz.Plan(n, 1)
res = torch.empty(plan.shard_residue_bytes() // 4, dtype=torch.int32, device="cuda")
out = torch.empty(n, dtype=torch.complex128, device="cuda")
y1 = torch.empty_like(x)
names = ["split_max", "split_digits", "col_fwd", "row_fused", "col_inv", "crt_finish"]


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps
    plan.profile(True)
    fn()
    torch.cuda.synchronize()
    prof = plan.profile_read()
    plan.profile(False)
    return t, prof


def shard():
    g = plan.shard_partial(x, 0, 1, res)
    plan.shard_finish(res, g, out)


for name, fn in [("shard N=1", shard), ("execute B=1", lambda: plan.forward(x, out=y1))]:
    t, prof = timed(fn)
    print(f"{name}: {t * 1000:.1f} us/transform")
    for k, v in prof.items():
        print(f"   {names[k] if isinstance(k, int) and k < len(names) else k}: {v}")
