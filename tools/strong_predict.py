"""Per-rank device time of the batch-sharded configs at N = 1, 2, 4, 8 (each rank's slice timed
alone on one GPU): predicts the strong-scaling speedup B / max_r t_r of bench.py --gpus N.
    python tools/strong_predict.py [c2 c3 c4 c5]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_29129_b200 as oz  # noqa: E402
import workloads  # noqa: E402
from paper_2603_29129_b200.dist import batch_slice  # noqa: E402

out = {}
for name in sys.argv[1:] or ["c2", "c3", "c4", "c5"]:
    cfg = workloads.CONFIGS[name]
    x_all = torch.from_numpy(workloads.config_input(cfg))
    res = {}
    for N in (1, 2, 4, 8):
        B = batch_slice(cfg.batch, 0, N)[1]
        x = x_all[:B].contiguous().cuda()
        plan = oz.Plan(cfg.n, B)
        o = torch.empty_like(x)
        back = torch.empty_like(x)
        for _ in range(4):
            plan.forward(x, out=o)
            if cfg.roundtrip:
                plan.inverse(o, out=back)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        reps = 10
        ev[0].record()
        for _ in range(reps):
            plan.forward(x, out=o)
            if cfg.roundtrip:
                plan.inverse(o, out=back)
        ev[1].record()
        torch.cuda.synchronize()
        res[N] = ev[0].elapsed_time(ev[1]) / reps
        del plan
    sp = {N: res[1] / res[N] for N in res}
    out[name] = {"ms_per_rank": res, "predicted_speedup": sp}
    print(name, json.dumps(out[name]), flush=True)
