#!/usr/bin/env python
"""bench.py -- fp64-accurate FFT via 32-bit NTTs (arXiv 2603.29129) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Metric (BASELINE.json): pseudo-GFLOP/s = transforms * 5 n log2 n / time, quoted at
n = 2^18 (config c3: batch 16 complex fp64 DFTs, m = 2^19).  A "step" is one pass
of the whole hot path (premultiply + split, 12 forward NTTs, NTT-domain
accumulation, 40 inverse NTTs, CRT, recombination, post-chirp) over the batch.

Multi-GPU (one process per GPU: torchrun, or `--gpus N` alone, which starts the N ranks
itself): the configured batch is sharded -- rank r transforms rows batch_slice(B, r, N) of
the same seeded input (SURVEY 8(e), strong scaling of the configured job); there is no
data-path collective; the timed region is bracketed by barriers, the reported time is the
max over ranks (all_reduce MAX of each rank's CUDA-event time) and value = B / that time.
After timing the rows are all-gathered and compared bit for bit with one GPU transforming
the whole batch ("bitwise_vs_n1").

--impl reference times the CPU oracle (oracle/, plain C, OpenMP over transforms)
on this box's host cores: the reference arm of this tier.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "fp64-accurate FFT GFLOP/s (5n·log2 n) at n=2^18; NTT HBM GB/s vs peak"
UNIT = "GFLOP/s"

# roofline denominators
MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK_GBS = 6650.0        # B200_PROFILING.md fallback
# Integer-pipe roofline, derived from unit counts and clocks: the ALU
# and FMA pipes each retire 64 lanes/clk/SM (B300_MICROARCH.md "rt_SMSP=2"; confirmed for
# IADD3, VIADDMNMX and IMAD on this pool's B200, IMAD.HI at half that rate,
# profiles/r01_microbench_bfly.txt).  A canonical Shoup butterfly needs IMAD.HI (2 slots)
# + 2 IMAD + 2 VIADDMNMX + 2 adds = 8 lane-slots of the 128 per clock -> 16 per SM per clock.
BFLY_PER_SM_CLK = 16
SMS = 148


def alu_peak_gbfly():
    mhz = 1965.0
    try:
        with open(MEASURED_PEAKS) as f:
            mhz = float(json.load(f).get("sm_max_mhz", mhz))
    except Exception:
        pass
    return BFLY_PER_SM_CLK * SMS * mhz * 1e6 / 1e9


ALU_BFLY_PEAK_GPS = alu_peak_gbfly()


def hbm_peak():
    try:
        with open(MEASURED_PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


def workload_desc(cfg):
    dist = {"uniform": "re/im uniform[-1,1)", "normal": "re/im standard normal",
            "signexp": "re/im sign*2^e, e in [-30,30]"}[cfg.dist]
    return (f"{cfg.name}: batch {cfg.batch} complex fp64 DFTs, n={cfg.n} (Bluestein m="
            f"{1 << math.ceil(math.log2(2 * cfg.n - 1))}), {dist}, seed {cfg.seed}")


def flops_per_transform(n):
    return 5.0 * n * math.log2(n)


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons (NVML) during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------- oracle timing
def time_oracle(cfg, ntrans, nthreads=0, reps=1):
    import oracle as O
    x = workloads.draw(cfg.dist, cfg.seed, cfg.batch, cfg.n, rows=slice(0, min(ntrans, cfg.batch)))
    if x.shape[0] < ntrans:  # sample larger than the batch: repeat rows
        x = np.ascontiguousarray(np.concatenate([x] * (ntrans // x.shape[0] + 1))[:ntrans])
    plan = O.Plan(cfg.n)
    ts, used = [], 1
    for _ in range(reps):
        t0 = time.perf_counter()
        y, used = plan.execute_batch(x, nthreads=nthreads)
        if cfg.roundtrip:
            plan.execute_batch(y, inverse=True, nthreads=nthreads)
        ts.append(time.perf_counter() - t0)
    dirs = 2 if cfg.roundtrip else 1
    return ts, used, x.shape[0] * dirs


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return  # other ranks exit 0 without work
    cores = host_cores()
    ntrans = min(cfg.batch, cores)
    for _ in range(args.warmup):
        time_oracle(cfg, ntrans)
    ts = []
    used = 1
    for _ in range(args.steps):
        t, used, units = time_oracle(cfg, ntrans)
        ts.append(t[0])
    tot = sum(ts)
    value = units * args.steps * flops_per_transform(cfg.n) / tot / 1e9
    t1, _, _ = time_oracle(cfg, 1, nthreads=1)  # single-thread time of one transform
    sample = (f"{ntrans} of the {cfg.batch} transforms of {cfg.name} per step "
              f"({'fwd+inv' if cfg.roundtrip else 'fwd'}), OpenMP over transforms")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64+u64", "data": "synthetic",
            "config": {"workload": workload_desc(cfg), "n": cfg.n, "batch": cfg.batch, "K": 3,
                       "L": 3, "impl": "CPU oracle (oracle/ozfft_oracle.c)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": "oracle",
                             "sample": sample,
                             "single_thread_s_per_transform": t1[0] / (2 if cfg.roundtrip else 1)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU arm
def run_single(args, cfg, rank, world, local_rank):
    """--mode single: ONE transform (row 0 of the config) sharded over the ranks by
    (prime, real convolution) units, one in-place NCCL all_gather_into_tensor of the
    inverse-NTT residues (8 g n words, g = the schedule's group count), then CRT +
    recombination on every rank.  Strong scaling; device
    time per step = max over ranks (CUDA events on the stream)."""
    import torch
    import paper_2603_29129_b200 as oz
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
    n = cfg.n
    x = torch.from_numpy(workloads.draw(cfg.dist, cfg.seed, cfg.batch, n, rows=slice(0, 1))).to(dev)
    plan = oz.Plan(n, 1, device=dev)
    stream = torch.cuda.current_stream(dev)

    residues = torch.empty(plan.shard_residue_bytes() // 4, dtype=torch.int32, device=dev)
    out = torch.empty(n, dtype=torch.complex128, device=dev)
    ag = []  # (start, end) events around the all-gather of each timed step
    gsz = [0]
    p2p = getattr(args, "p2p", False)
    peers = [residues.data_ptr()]
    if p2p and world > 1:  # every rank's exchange buffer mapped into this process (CUDA IPC)
        handles = [None] * world
        dist.all_gather_object(handles, oz.ipc_handle(residues))
        peers = [residues.data_ptr() if r == rank else oz.ipc_open(handles[r], dev) for r in range(world)]
    token = torch.zeros(1, device=dev)

    def step(record=False):
        if p2p:
            # the producing kernels store every residue into every rank's buffer; a one-word
            # all-reduce on the stream is the device-side barrier before the finish
            g = plan.shard_partial_p2p(x, rank, world, peers)
            gsz[0] = g
            if world > 1:
                if record:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                dist.all_reduce(token)
                if record:
                    e1.record(stream)
                    ag.append((e0, e1))
            return plan.shard_finish(residues, g, out)
        g = plan.shard_partial(x, rank, world, residues)
        gsz[0] = g
        if world > 1:
            buf = residues[:8 * g * n]
            per = buf.numel() // world
            if record:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            dist.all_gather_into_tensor(buf, buf[rank * per:(rank + 1) * per])  # in place
            if record:
                e1.record(stream)
                ag.append((e0, e1))
        return plan.shard_finish(residues, g, out)

    for _ in range(max(args.warmup, 3)):
        y = step()
    torch.cuda.synchronize(dev)
    ref = plan.forward(x)
    assert torch.equal(y.view(1, n), ref), "sharded transform differs from the one-GPU execute"
    if dist:
        dist.barrier()
    launches0 = oz.kernel_launches()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    torch.cuda.synchronize(dev)
    for i in range(args.steps):
        ev[i][0].record(stream)
        step(record=True)
        ev[i][1].record(stream)
    torch.cuda.synchronize(dev)
    t_ms = sum(a.elapsed_time(b) for a, b in ev)
    ag_ms = sum(a.elapsed_time(b) for a, b in ag)
    if dist:
        t = torch.tensor([t_ms, ag_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms, ag_ms = float(t[0].item()), float(t[1].item())
    if rank == 0:
        nbytes = plan.shard_residue_bytes(gsz[0])
        ag_per = ag_ms / args.steps
        busbw = (nbytes * (world - 1) / world) / (ag_per * 1e-3) / 1e9 if ag_per > 0 else None
        if p2p:
            allgather = {"ms_per_step": ag_per, "bytes": nbytes, "groups": gsz[0],
                         "note": "peer-memory exchange fused into the inverse-NTT epilogue (stores "
                                 "into every rank's buffer through CUDA IPC mappings); ms_per_step "
                                 "is the one-word all-reduce used as the barrier after it"}
        else:
            allgather = None
        allgather = allgather or {"ms_per_step": ag_per, "bytes": nbytes, "groups": gsz[0],
                     "busbw_GBs": busbw,
                     "frac_of_peer_copy_770GBs": busbw / 770.0 if busbw else None,
                     "note": "in-place NCCL all_gather_into_tensor of the inverse-NTT residues "
                             "[8 units][g][n], CUDA events on the stream, max over ranks; busBW = "
                             "bytes (N-1)/N / time; reference: 770 GB/s measured peer copy "
                             "(B200_PROFILING.md)"}
        line = {"metric": METRIC, "value": args.steps * flops_per_transform(n) / (t_ms * 1e-3) / 1e9,
                "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
                "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "u32", "data": "synthetic",
                "config": {"workload": f"single-transform variant of {cfg.name}: transform 0, n={n}, "
                                       f"units (prime, conv) split over {world} rank(s), "
                                       + ("residues stored into every rank's buffer by the producing "
                                          "kernels (peer memory)" if p2p else
                                          "one NCCL all-gather of the residues") + " before CRT",
                           "n": n, "m": plan.m, "parallelism": f"unit-sharded x{world}",
                           "residue_bytes_gathered": nbytes if world > 1 else 0},
                "gpu_launches": int(oz.kernel_launches() - launches0),
                "allgather": allgather if world > 1 else None}
        print(json.dumps(line), flush=True)


class Coll:
    """The collectives of the batch-sharded bench, in one fixed order on every rank (an idle
    rank -- more ranks than transforms -- issues the same calls with empty data)."""

    def __init__(self, world, dev):
        import torch
        self.world, self.dev, self.torch = world, dev, torch
        self.dist = None
        if world > 1:
            import torch.distributed as dist
            self.dist = dist
            if dist.get_backend() == "gloo":  # (test knob --backend gloo: host tensors)
                self.dev = torch.device("cpu")

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, v):
        if not self.dist:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def gather_rows(self, y, total, n):
        """All ranks' output rows (complex128 [count_r, n]) -> [total, n] on every rank, in
        batch order (rank r's rows are batch_slice(total, r, world))."""
        torch = self.torch
        if not self.dist:
            return y
        from paper_2603_29129_b200.dist import batch_slice
        cmax = -(-total // self.world)
        pad = torch.zeros(cmax, n, dtype=torch.complex128, device=self.dev)
        if y is not None and y.shape[0]:
            pad[:y.shape[0]] = y.to(self.dev)
        allr = torch.empty(self.world * cmax, n, dtype=torch.complex128, device=self.dev)
        self.dist.all_gather_into_tensor(torch.view_as_real(allr), torch.view_as_real(pad))
        rows = [allr[r * cmax: r * cmax + batch_slice(total, r, self.world)[1]] for r in range(self.world)]
        return torch.cat(rows).to(y.device if y is not None else self.dev)


def rank_input(cfg, rank, world):
    """Rank r's contiguous slice of the config's ONE seeded batch (the batch of
    independent transforms is sharded, B / N per rank; every rank draws the same bytes and
    keeps its rows, so the N-GPU job transforms exactly the N = 1 input)."""
    from paper_2603_29129_b200.dist import batch_slice
    start, cnt = batch_slice(cfg.batch, rank, world)
    x = workloads.config_input(cfg)
    return start, cnt, np.ascontiguousarray(x[start:start + cnt])


def run_ours(args, cfg, rank, world, local_rank):
    import torch
    import paper_2603_29129_b200 as oz
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
    Bg, n = cfg.batch, cfg.n
    # strong scaling over the configured batch: rank r transforms rows [start, start + B)
    start, B, x_np = rank_input(cfg, rank, world)
    coll = Coll(world, dev)
    if B == 0:  # more ranks than transforms (c1 at N > 1): join the collectives only
        coll.barrier()
        coll.max(0.0)
        coll.barrier()
        coll.barrier()
        coll.max(0.0)
        coll.gather_rows(None, Bg, n)
        if cfg.roundtrip:
            coll.gather_rows(None, Bg, n)
        return
    x = torch.from_numpy(x_np).to(dev)
    plan = oz.Plan(n, B, device=dev, conv=args.conv, accum=args.accum, precision=args.precision)
    out = torch.empty_like(x)
    back = torch.empty_like(x) if cfg.roundtrip else None
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step():
        plan.forward(x, out=out)
        if cfg.roundtrip:
            plan.inverse(out, out=back)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize(dev)
    coll.barrier()
    # timed region: the production path (no stage timers; plans with batch*m <= 2^25 replay a
    # CUDA graph, captured during the warm-up)
    launches0 = oz.kernel_launches()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    sampler = ClockSampler(local_rank)
    torch.cuda.synchronize(dev)
    with sampler:
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize(dev)
    launches = oz.kernel_launches() - launches0
    per_step = sorted(a.elapsed_time(b) for a, b in ev)
    step_ms = {"median": statistics.median(per_step), "min": per_step[0], "max": per_step[-1],
               "note": "rank-local CUDA-event time of each timed step (rank 0)"}
    # second timed pass of the same steps with the per-stage CUDA-event timers (stream-
    # ordered on the execute stream): the stage breakdown and the roofline's kernel times
    plan.profile(True)
    for i in range(args.steps):
        flush.zero_()
        step()
    torch.cuda.synchronize(dev)
    prof = plan.profile_read()
    plan.profile(False)
    t_ms = coll.max(sum(a.elapsed_time(b) for a, b in ev))  # max over ranks
    coll.barrier()
    stats = plan.stats()
    dirs = 2 if cfg.roundtrip else 1
    total_transforms = Bg * dirs * args.steps
    value = total_transforms * flops_per_transform(n) / (t_ms * 1e-3) / 1e9

    # ---- end to end through the C ABI with HOST buffers (pinned), copies inside the region
    xh = torch.from_numpy(x_np).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    zh = torch.empty_like(xh).pin_memory() if cfg.roundtrip else None

    def e2e_step():
        plan.execute_host(xh, -1, out_host=yh)
        if cfg.roundtrip:
            plan.execute_host(yh, +1, out_host=zh)

    for _ in range(2):
        e2e_step()
    e2e_steps = max(3, min(args.steps, 10))
    coll.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    torch.cuda.synchronize(dev)
    e2e_s = coll.max(time.perf_counter() - t0)
    e2e_val = Bg * dirs * e2e_steps * flops_per_transform(n) / e2e_s / 1e9
    io_bytes = Bg * n * 16 * dirs

    # ---- the N-rank outputs against one GPU transforming the whole batch (rank 0)
    step()
    torch.cuda.synchronize(dev)
    y_all = coll.gather_rows(out, Bg, n)
    b_all = coll.gather_rows(back, Bg, n) if cfg.roundtrip else None
    bitwise = None
    if world > 1 and rank == 0:
        xf = torch.from_numpy(workloads.config_input(cfg)).to(dev)
        pf = oz.Plan(n, Bg, device=dev, conv=args.conv, accum=args.accum, precision=args.precision)
        yf = pf.forward(xf)
        bitwise = bool(torch.equal(yf, y_all.to(dev)))
        if cfg.roundtrip:
            bitwise = bitwise and bool(torch.equal(pf.inverse(yf), b_all.to(dev)))
        del pf, xf, yf

    if rank != 0:
        return
    # ---- roofline of the dominant stage kernel (live CUDA-event times of the timed region)
    m = plan.m
    logR, logC = plan.log2_rows, plan.log2_cols
    execs = args.steps * dirs
    fwd_vec = stats["fwd_ntts"]  # forward NTT vectors of the last execute (whole batch)
    inv_vec = stats["inv_ntts"]  # inverse NTT vectors (2 per Alg.8 group)
    per_exec = {  # (bytes, butterflies) per execute over the batch -- DESIGN.md "Algorithmic work"
        # x (16 n B per transform) per level; the chirp (16 n B) is shared by the batch
        "split_max": (plan.K * (16 * n * B + 16 * n), 0) if prof["split_digits"][1]
        else (16 * n * B + 16 * n + 24 * n * B, 0),  # n <= 2^15: one cluster launch (x once, digits)
        "split_digits": (16 * n * B + 16 * n + 24 * n * B, 0),
        "col_fwd": (fwd_vec * 4 * (n + m), fwd_vec * (m // 2) * logR),
        "row_fused": (fwd_vec * 4 * m + inv_vec * 4 * m, (fwd_vec + inv_vec) * (m // 2) * logC),
        "col_inv": (inv_vec * 4 * (m + n), inv_vec * (m // 2) * logR),
        "crt_finish": (inv_vec * 4 * n + 32 * n * B, 0),
    }
    nsums = 2 if args.accum == "image" else 4  # DD sums per transform: Re, Im (f2) or rr, ii, ir, ri
    if logR > 0:  # fused inverse column pass + CRT + DD accumulation; finish reads the DD sums
        per_exec["col_inv"] = (inv_vec * 4 * m + 16 * nsums * n * B, inv_vec * (m // 2) * logR)
        per_exec["crt_finish"] = ((16 * nsums + 16) * n * B + 16 * n, 0)  # sums + out, chirp once
    hbm, hbm_kind = hbm_peak()
    stages = {}
    for s, (ms, cnt) in prof.items():
        if cnt == 0:
            continue
        ms_per_launch = ms / cnt
        byts, bfly = per_exec[s]
        launches_per_exec = cnt / execs
        byts /= launches_per_exec
        bfly /= launches_per_exec
        gbs = byts / (ms_per_launch * 1e-3) / 1e9
        gbf = bfly / (ms_per_launch * 1e-3) / 1e9
        stages[s] = {"ms_per_launch": ms_per_launch, "share": ms / sum(v[0] for v in prof.values()),
                     "GB_s": gbs, "frac_hbm": gbs / hbm, "Gbfly_s": gbf,
                     "frac_alu": gbf / ALU_BFLY_PEAK_GPS, "launches": cnt}
    dom = max(stages, key=lambda s: stages[s]["share"])
    d = stages[dom]
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            with open(tfile) as f:
                traffic = json.load(f).get(cfg.name, {}).get(dom)
        except Exception:
            traffic = None
    if d["frac_alu"] >= d["frac_hbm"]:
        roof = {"bound": "alu", "achieved": d["Gbfly_s"], "peak": ALU_BFLY_PEAK_GPS,
                "unit": "Gbutterfly/s", "frac": d["frac_alu"], "traffic": traffic,
                "peak_kind": "derived: 16 Shoup butterflies/clk/SM (64-lane ALU + 64-lane FMA "
                             "pipes, 8 lane-slots per butterfly) x 148 SMs x sm_max clock; "
                             "in-register radix-16 measured 13.1/clk/SM (tools/microbench_bfly.cu)",
                "kernel": dom, "hbm_GB_s": d["GB_s"], "hbm_frac": d["frac_hbm"],
                "hbm_frac_of_8TBs_spec": d["GB_s"] / 8000.0}
    else:
        roof = {"bound": "hbm", "achieved": d["GB_s"], "peak": hbm, "unit": "GB/s",
                "frac": d["frac_hbm"], "traffic": traffic, "peak_kind": hbm_kind + " (MEASURED_PEAKS.json)",
                "kernel": dom, "alu_Gbfly_s": d["Gbfly_s"], "alu_frac": d["frac_alu"]}

    # ---- CPU baseline: the oracle on a bounded sample, rank 0 at N = 1 only
    cpu = None
    if world == 1 and not args.no_cpu:
        cores = host_cores()
        ntr = min(cfg.batch, cores)
        ts, used, units = time_oracle(cfg, ntr)
        cpu = {"value": units * flops_per_transform(n) / ts[0] / 1e9, "unit": UNIT, "cores": used,
               "kind": "oracle",
               "sample": f"{ntr} transforms of {cfg.name} ({'fwd+inv' if cfg.roundtrip else 'fwd'}), "
                         f"{ts[0]:.1f} s wall, OpenMP over transforms"}
    # ---- side measurements, same protocol, reported beside the headline (which follows the
    # north star: m >= 2n-1, the paper's four real convolutions):
    #   f1_cyclic: the paper's N = n cyclic Bluestein for power-of-two n, output
    #              bitwise equal to the headline's (tests/test_gpu_cyclic.py);
    #   f2_image:  complex-image accumulation (beyond the paper; own oracle mode,
    #              tests/test_gpu_image.py), padded and, for power-of-two n, cyclic.
    def side(conv, accum, precision="dd"):
        pc = oz.Plan(n, B, device=dev, conv=conv, accum=accum, precision=precision)

        def cstep():
            pc.forward(x, out=out)
            if cfg.roundtrip:
                pc.inverse(out, out=back)

        for _ in range(max(args.warmup, 3)):
            cstep()
        cev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        torch.cuda.synchronize(dev)
        for i in range(args.steps):
            flush.zero_()
            cev[i][0].record(stream)
            cstep()
            cev[i][1].record(stream)
        torch.cuda.synchronize(dev)
        c_ms = sum(a.elapsed_time(b) for a, b in cev)
        st = pc.stats()
        r = {"value": total_transforms * flops_per_transform(n) / (c_ms * 1e-3) / 1e9,
             "unit": UNIT, "ms_per_step": c_ms / args.steps, "m": pc.m, "alpha": pc.alpha,
             "conv": conv, "accum": accum, "precision": precision,
             "ntt_split": f"m = 2^{pc.log2_rows} x 2^{pc.log2_cols}",
             "ntts_per_transform": (st["fwd_ntts"] + st["inv_ntts"]) / B}
        del pc
        return r

    pow2 = n > 1 and n & (n - 1) == 0
    cyc = img = imgc = tsl = None
    if (args.conv == "padded" and args.accum == "real" and args.precision == "dd"
            and not args.no_extra and world == 1):  # side lines at N = 1 only
        if pow2:
            cyc = side("cyclic", "real")
            cyc["note"] = "paper's N = n cyclic Bluestein (P:238-241); bitwise equal to the headline"
        img = side("padded", "image")
        img["note"] = "complex-image accumulation (SURVEY f2; beyond the paper; own oracle mode)"
        if pow2:
            imgc = side("cyclic", "image")
        tsl = side("padded", "real", "ts")
        tsl["note"] = "the paper's triple-single working precision (SURVEY f4)"
    clocks = sampler.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": t_ms / args.steps, "step_ms": step_ms,
        "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": workload_desc(cfg), "n": n, "m": m, "batch_per_gpu": B,
                   "global_batch": Bg, "K": plan.K, "L": plan.L, "alpha": plan.alpha,
                   "ntt_split": f"m = 2^{logR} x 2^{logC}", "parallelism": f"batch-sharded x{world}",
                   "directions": "fwd+inv" if cfg.roundtrip else "fwd",
                   "l2": "flushed between timed steps (512 MiB write outside the events)",
                   "inputs": "config recipe; rank r transforms rows batch_slice(B, r, N) of it",
                   "io_dtype": "complex128", "conv": args.conv, "accum": args.accum,
                   "precision": args.precision},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": io_bytes,
                "d2h_bytes_per_step": io_bytes, "steps": e2e_steps},
        "gpu_launches": int(launches),
        "bitwise_vs_n1": bitwise,
        "test_knobs": ({"backend": args.backend, "one_device": True} if args.one_device else None),
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "stages": stages,
        "stages_note": "per-stage CUDA events (execute stream) from a second pass of the same "
                       "steps with the stage timers on; the timed region itself runs without them",
        "ntt_counts_per_transform": {"fwd": stats["fwd_ntts"] / B, "inv": stats["inv_ntts"] / B,
                                     "cached": stats["cached_ntts"]},
        "f1_cyclic": cyc,
        "f2_image": img,
        "f1_f2_cyclic_image": imgc,
        "f4_ts": tsl,
    }
    print(json.dumps(line), flush=True)


def _spawned_rank(local_rank, argv, world, port):
    """Rank entry of `bench.py --gpus N` started without torchrun (one process per GPU)."""
    os.environ.update({"RANK": str(local_rank), "LOCAL_RANK": str(local_rank),
                       "WORLD_SIZE": str(world), "MASTER_ADDR": "127.0.0.1",
                       "MASTER_PORT": str(port)})
    sys.argv = argv
    main()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="ranks (one per GPU); under torchrun it must equal WORLD_SIZE, "
                         "without torchrun bench.py starts the N ranks itself")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(workloads.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle cpu_baseline leg")
    ap.add_argument("--conv", default="padded", choices=["padded", "cyclic"],
                    help="Bluestein length: m >= 2n-1 (north star) or m = n (P:238-241)")
    ap.add_argument("--p2p", action="store_true",
                    help="--mode single: the residue exchange fused into the producing kernels "
                         "(peer-memory stores through CUDA IPC mappings) instead of an NCCL all-gather")
    ap.add_argument("--mode", default="batch", choices=["batch", "single"],
                    help="batch: the configured batch sharded over the ranks (the headline); "
                         "single: one transform sharded over the ranks by (prime, conv) units "
                         "with an NCCL all-gather (SURVEY 8(e))")
    ap.add_argument("--precision", default="dd", choices=["dd", "ts"],
                    help="double-double O(n) steps (default) or the paper's triple-single (f4)")
    ap.add_argument("--accum", default="real", choices=["real", "image"],
                    help="four real convolutions (the paper) or complex images (SURVEY f2)")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the f1_cyclic / f2_image side measurements")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo + --one-device: a test of the N-rank "
                         "batch path on a one-GPU box; its kernels never wait on each other)")
    ap.add_argument("--one-device", action="store_true",
                    help="every rank on cuda:0 (test knob; timings are not N-GPU numbers)")
    args = ap.parse_args()
    cfg = workloads.CONFIGS[args.config]
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus and args.gpus > 1:
        import socket
        import torch.multiprocessing as mp
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        mp.start_processes(_spawned_rank, args=(list(sys.argv), args.gpus, port),
                           nprocs=args.gpus, join=True, start_method="spawn")
        return
    world = int(env_world or "1")
    if args.gpus is not None and args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = 0 if args.one_device else int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if args.backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.mode == "single":
            run_single(args, cfg, rank, world, local_rank)
        else:
            run_ours(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
