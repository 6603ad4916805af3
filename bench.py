#!/usr/bin/env python
"""Benchmark of the BAL inexact Newton-PCG time step (arXiv 2407.00046) on B200.

Metric (BASELINE.json): "seconds/frame & PCG iters/s at 1.76M tets; BSR SpMV HBM GB/s vs peak".
Workload: the C4 puffer-balls-on-chain-net scene (configs[3], ~1.75M tets, dt = 1/30 s) in its
contact-rich start (scenes.make_puffer_net(settled=True): connectors hanging on the net, balls
resting above it; ~2.6e5 active constraints, the paper's 228K avg / 292K max).  A C4
frame takes hundreds of inexact-Newton iterations of thousands of PCG iterations each (the paper
reports 156.8 Newton iterations and 427 s per frame on its GPU), so one bench step is ONE
inexact-Newton iteration of Alg. 1 -- every row of SURVEY §8(a) once: constraint sets, elastic /
contact / friction stencils, atomic-free assembly, warm start, global PCG, CCD line search, AL
updates (a1 at every frame start) -- and the simulation continues across steps, frame after frame.
`value` = global PCG iterations per second of the whole job (all phases in the denominator; N
ranks each advance their own replica: weak scaling, no data-path collective).  Seconds per frame
are reported when a frame completes inside the timed region, and as ms/Newton x the Newton
iterations per frame of a recorded long run (profiles/c4_frames.json) otherwise, labelled so.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c4|c4-drop|c1|c5]

Headline fields of the line: ms_per_newton (all phases of one Newton iteration), the active
constraint counts of the timed iterations, and seconds_per_frame when a frame completes inside the
timed region (else the whole-frame runs measured separately, cited by file).  `value` (PCG iters/s
over whole Newton iterations) is the metric's second component.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "seconds/frame & PCG iters/s at 1.76M tets; BSR SpMV HBM GB/s vs peak"
UNIT = "PCG iters/s"
# PCG iterations per Newton iteration of the GPU path on the bench workload, read from the last
# committed bench line (profiles/bench_r02_c4.json) so the reference (oracle) arm's step does the
# same work; fallback: the App. B cap the contact-rich start hits (20,000)
C4_PCG_PER_NEWTON_FALLBACK = 20000.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=["c4", "c4-drop", "c1", "c5"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fp32-matrix", action="store_true",
                    help="NEXT-3 variant: SpMV streams FP32-rounded static blocks (FP64 arithmetic)")
    return ap.parse_args()


def make_scene(cfg):
    import scenes
    if cfg == "c1":
        return scenes.make_cubes(1), "C1 two stacked soft cubes (1.5K tets), dt=1/30 s"
    if cfg == "c5":
        return scenes.make_puffer_tiles(5), "C5 3x2 replicated puffer-net tiles (~10.5M tets) on ONE GPU, dt=1/30 s"
    if cfg == "c4-drop":
        return scenes.make_puffer_net(seed=4), "C4 puffer balls dropped on chain-net (~1.7M tets, few contacts), dt=1/30 s"
    return (scenes.make_puffer_net(seed=4, settled=True),
            "C4 puffer balls on chain-net, contact-rich start (~1.7M tets, ~2.6e5 constraints), dt=1/30 s")


def gpu_pcg_per_newton(cfg):
    f = os.path.join(ROOT, "profiles", f"bench_r02_{cfg}.json")
    try:
        with open(f) as fh:
            return float(json.load(fh)["pcg_iters_per_newton"]), f"GPU run's mean ({os.path.relpath(f, ROOT)})"
    except Exception:  # noqa: BLE001
        return C4_PCG_PER_NEWTON_FALLBACK, "App. B cap (no committed GPU line)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([s.strip() for s in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and "Active" in r[3 + i]
                          and "Not" not in r[3 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def job_throughput(local_seconds, units_per_rank, world, device, shared=False):
    """Max of the ranks' timed-region seconds (the job time) and the whole-job throughput
    (units processed by all ranks / job time).  One all_reduce(MAX) when world > 1.  shared: the
    ranks cooperate on ONE problem (partitioned solve), so the job's units are one rank's count."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(local_seconds)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    s = float(t.item())
    return s, (1 if shared else world) * units_per_rank / s


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# --------------------------------------------------------------------------- oracle timing
def oracle_sample(sc, newton_per_frame, pcg_per_newton, budget_tets=20000, seed=0):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload and scale to s/frame:
    one Newton iteration = elastic AD stencils + eigh projection over all tets (timed on a random
    sample of `budget_tets` tets, scaled by T) + `pcg_per_newton` PCG iterations (SpMV timed on the
    CSR assembled from the sampled stencils, scaled by nnz; vector updates timed at full size)."""
    import scipy.sparse as sp

    from oracle.energy import nh_stencils
    from oracle.mesh import precompute
    from oracle.projection import project_eigh

    threads = int(os.environ.get("OMP_NUM_THREADS", "0") or 0) or (os.cpu_count() or 1)
    m = precompute(sc)
    rng = np.random.default_rng(seed)
    T = len(m.tets)
    sel = rng.choice(T, size=min(budget_tets, T), replace=False)
    sub = type(m)(**{**m.__dict__, "tets": m.tets[sel], "Dm_inv": m.Dm_inv[sel], "vol": m.vol[sel],
                     "mu": m.mu[sel], "lam": m.lam[sel], "arap": m.arap[sel]})
    x = np.asarray(sc["x0"], np.float64)
    t0 = time.perf_counter()
    _v, _g, H = nh_stencils(x, sub)
    P, _ = project_eigh(H)
    t_st = time.perf_counter() - t0
    t_asm = t_st * T / len(sel)
    dof = (3 * sub.tets[:, :, None] + np.arange(3)[None, None]).reshape(-1, 12)
    rows = np.repeat(dof, 12, axis=1).ravel()
    cols = np.tile(dof, (1, 12)).ravel()
    n3 = 3 * len(x)
    A = sp.coo_matrix((P.ravel(), (rows, cols)), shape=(n3, n3)).tocsr()
    v = rng.normal(size=n3)
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        A @ v
    t_spmv_s = (time.perf_counter() - t0) / reps
    # full-size static matrix nnz: 9 * (N + 2E); E from unique tet edges
    e = np.concatenate([m.tets[:, [a, b]] for a in range(4) for b in range(a + 1, 4)])
    E = len(np.unique(np.sort(e, axis=1), axis=0))
    nnz_full = 9 * (len(x) + 2 * E)
    t_spmv = t_spmv_s * nnz_full / max(A.nnz, 1)
    t0 = time.perf_counter()
    for _ in range(reps):  # ~12 vector passes of textbook PCG
        a = v + 0.5 * v
        b = a - 0.25 * v
        float(a @ b)
        float(b @ b)
        c = a * 1.0001
        float(c @ a)
    t_vec = (time.perf_counter() - t0) / reps * 2.0
    t_pcg = t_spmv + t_vec
    t_newton = t_asm + pcg_per_newton * t_pcg
    s_frame = newton_per_frame * t_newton
    desc = (f"oracle timed on {len(sel)} sampled tets (AD + eigh, scaled x{T / len(sel):.0f}) and a CSR SpMV "
            f"of their stencils (scaled by nnz to the full static matrix) + full-size vector passes; frame = "
            f"{newton_per_frame:.1f} Newton x (assembly + {pcg_per_newton:.0f} PCG iterations), counts from the "
            f"GPU path on the same scene (extrapolated, not a measured frame)")
    return s_frame, threads, desc, dict(t_assembly_s=t_asm, t_pcg_iter_s=t_pcg, sample_s=t_st + t_spmv_s * reps)


# --------------------------------------------------------------------------- arms
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sc, wl = make_scene(args.config)
    ppn, ppn_src = gpu_pcg_per_newton(args.config) if args.config.startswith("c4") else (100.0, "fixed")
    vals = []
    t_all = time.perf_counter()
    info = {}
    for _ in range(max(args.warmup, 0)):
        oracle_sample(sc, 1.0, ppn, budget_tets=2000)
    threads, desc = 0, ""
    for k in range(args.steps):
        _s, threads, desc, info = oracle_sample(sc, 1.0, ppn, budget_tets=5000, seed=k)
        vals.append(info["t_assembly_s"] + ppn * info["t_pcg_iter_s"])
    s_newton = float(np.mean(vals))
    v = ppn / s_newton
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * s_newton, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl, "tets": int(len(sc["tets"])), "nodes": int(len(sc["rest_x"])),
                       "step": "one inexact-Newton iteration of Alg. 1"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": desc + f"; one step = assembly + {ppn:.0f} PCG iterations ({ppn_src}), "
                                              f"extrapolated"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "detail": {**info, "wall_s": time.perf_counter() - t_all}}
    print(json.dumps(line), flush=True)


class FrameRunner:
    """Advances the simulation one inexact-Newton iteration (= one bench step: every §8(a) row
    a2-a11 once; a1 at each frame start) at a time through bal_frame_begin/iterate/finish,
    starting the next frame whenever one converges.  Keeps running totals of the library's
    per-frame counters."""

    def __init__(self, bal, ctx, x, v):
        import torch
        self.bal, self.ctx = bal, ctx
        self.x, self.v = x, v
        self.xn, self.vn = torch.empty_like(x), torch.empty_like(v)
        self.done = {"pcg_iters": 0, "newton_iters": 0, "ws_iters": 0, "ms_collision": 0.0, "ms_assembly": 0.0,
                     "ms_pcg": 0.0, "ms_linesearch": 0.0, "max_constraints": 0}
        self.frames = []  # (ms_total, newton_iters, pcg_iters) of completed frames
        self.unconverged = 0
        self.nA = []  # |A| of every Newton iteration run (decision trace)
        bal.bal_frame_begin(ctx, self.x, self.v)

    def totals(self):
        cur = self.bal.bal_frame_stats(self.ctx)
        t = dict(self.done)
        for k in t:
            if k == "max_constraints":
                t[k] = max(t[k], cur[k])
            else:
                t[k] += cur[k]
        return t

    def step(self):
        try:
            conv = self.bal.bal_frame_iterate(self.ctx, 1)
        except self.bal.BalError as e:  # Newton cap (BAL_E_NOT_CONVERGED): the frame ends unconverged
            if e.status != -4:
                raise
            self.unconverged += 1
            conv = True
        tr = self.bal.bal_get_trace(self.ctx, max_records=4096)
        if tr:
            self.nA.append(int(tr[-1]["nA"]))
        if conv:
            st = self.bal.bal_frame_finish(self.ctx, self.xn, self.vn, allow_unconverged=True)
            for k in self.done:
                self.done[k] = max(self.done[k], st[k]) if k == "max_constraints" else self.done[k] + st[k]
            self.frames.append((st["ms_total"], st["newton_iters"], st["pcg_iters"]))
            self.x, self.xn = self.xn, self.x
            self.v, self.vn = self.vn, self.v
            self.bal.bal_frame_begin(self.ctx, self.x, self.v)


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    import paper_2407_00046_b200 as bal

    sc, wl = make_scene(args.config)
    # N > 1: the partitioned solve of SURVEY §8(e) (vertex-domain row ranges, NCCL halo of p before
    # every SpMV + one all-reduce per PCG iteration; strong scaling of the one C4 problem).
    # BAL_BENCH_REPLICAS=1: N independent replicas instead (weak scaling, no data-path collective).
    replicas = world > 1 and os.environ.get("BAL_BENCH_REPLICAS") == "1"
    flags = bal.BAL_FP32_MATRIX if args.fp32_matrix else 0
    shared = world > 1 and not replicas
    if shared:
        obj = [bal.bal_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = bal.bal_init(sc, device=local, rank=rank, world=world, nccl_id=obj[0], flags=flags)
    else:
        ctx = bal.bal_init(sc, device=local, flags=flags)
    stream = torch.cuda.current_stream(dev)
    bal.bal_set_stream(ctx, stream)
    x = torch.as_tensor(sc["x0"].ravel(), device=dev)
    v = torch.as_tensor(sc["v0"].ravel(), device=dev)
    run = FrameRunner(bal, ctx, x, v)
    for _ in range(args.warmup):
        run.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    spmv0 = bal.bal_spmv_counters(ctx)
    nA0 = len(run.nA)
    launches0 = ctx.kernel_launches
    tot0 = run.totals()
    nf0 = len(run.frames)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            run.step()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = e0.elapsed_time(e1)
    launches = ctx.kernel_launches - launches0
    spmv1 = bal.bal_spmv_counters(ctx)
    tot1 = run.totals()
    d = {k: tot1[k] - tot0[k] for k in tot1 if k != "max_constraints"}
    pcg = d["pcg_iters"]
    newton = d["newton_iters"]
    s_max, pcg_per_s = job_throughput(ms / 1000.0, pcg, world, dev, shared)
    ms_max = 1000.0 * s_max
    new_frames = run.frames[nf0:]
    # SpMV roofline from the library's CUDA events around every SpMV launch in the timed region
    d_ms = spmv1["ms"] - spmv0["ms"]
    d_n = spmv1["launches"] - spmv0["launches"]
    d_alg = spmv1["bytes_alg"] - spmv0["bytes_alg"]
    d_mov = spmv1["bytes_moved"] - spmv0["bytes_moved"]
    peak, peak_src = measured_peaks()
    spmv_us = 1000.0 * d_ms / max(d_n, 1)
    achieved = (d_alg / max(d_n, 1)) / (spmv_us * 1e-6) / 1e9 if d_n else None
    moved_gbs = (d_mov / max(d_n, 1)) / (spmv_us * 1e-6) / 1e9 if d_n else None
    # ncu DRAM bytes per launch of the SpMV on this workload (one `ncu --set full` capture, committed
    # per config under profiles/; null when none was taken for this config)
    traffic, traffic_src = None, None
    tf = os.path.join(ROOT, "profiles", f"spmv_traffic_{args.config}.json")
    if os.path.exists(tf):
        with open(tf) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
        traffic_src = os.path.relpath(tf, ROOT)
    # SURVEY d.1 (b): PCG microbenchmark on the live (last assembled) C4 system: 1,000 global PCG
    # iterations, termination disabled, CUDA events (outside the timed region)
    pcg_micro = None
    try:
        b = torch.randn(x.numel(), dtype=torch.float64, device=dev)
        xo = torch.empty_like(b)
        z0 = torch.zeros_like(b)
        bal.bal_pcg(ctx, b, z0, xo, warm_start=0, rel_tol=0.0, stall_window=0, max_iters=50)  # warm-up
        m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        m0.record(stream)
        sm = bal.bal_pcg(ctx, b, z0, xo, warm_start=0, rel_tol=0.0, stall_window=0, max_iters=1000)
        m1.record(stream)
        torch.cuda.synchronize()
        pcg_micro = {"iters": int(sm["iters"]), "ms": m0.elapsed_time(m1),
                     "iters_per_s": 1000.0 * sm["iters"] / m0.elapsed_time(m1)}
    except Exception as ex:  # noqa: BLE001 -- reported, never fatal for the main line
        pcg_micro = {"error": str(ex)}
    # e2e through the public C ABI with HOST buffers: bal_step_host (x_t, v_t host -> device, the
    # time step, x_{t+1}, v_{t+1} device -> host inside the call) on a context whose Newton cap is
    # E2E_NEWTON iterations (BAL_E_NOT_CONVERGED returns the last accepted iterate and the stats),
    # timed on the host around the call
    e2e = None
    if not args.no_e2e:
        E2E_NEWTON = 2
        prm = dict(sc["params"])
        prm["max_newton"] = E2E_NEWTON
        if shared:
            obj = [bal.bal_nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            ctx2 = bal.bal_init(sc, device=local, params=prm, rank=rank, world=world, nccl_id=obj[0], flags=flags)
        else:
            ctx2 = bal.bal_init(sc, device=local, params=prm, flags=flags)
        xh = run.x.detach().cpu().numpy().copy()
        vh = run.v.detach().cpu().numpy().copy()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        _xn, _vn, st2 = bal.bal_step_host(ctx2, xh, vh, allow_unconverged=True)
        el = time.perf_counter() - t0
        _s, e2e_v = job_throughput(el, st2["pcg_iters"], world, dev, shared)
        nb = 3 * 8 * len(sc["rest_x"])
        e2e = {"value": e2e_v, "unit": UNIT, "h2d_bytes_per_step": 2 * nb, "d2h_bytes_per_step": 2 * nb,
               "newton_iters": st2["newton_iters"], "pcg_iters": st2["pcg_iters"], "seconds": el,
               "note": f"bal_step_host (host x_t, v_t in; x_t+1, v_t+1 out) with the Newton cap at {E2E_NEWTON}, "
                       "from the state the timed region ended in"}
        del ctx2
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    ppn = pcg / max(newton, 1)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        _s, threads, desc, info = oracle_sample(sc, 1.0, ppn)
        s_newton_cpu = info["t_assembly_s"] + ppn * info["t_pcg_iter_s"]
        cpu = {"value": ppn / s_newton_cpu, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": desc + f"; one step = assembly + {ppn:.0f} PCG iterations (the GPU run's mean), "
                                f"extrapolated"}
    ms_newton = ms_max / max(newton, 1)
    nA_t = run.nA[nA0:]
    # whole-frame runs of this workload measured separately (tools/c4_frames.py, committed under
    # profiles/ as <config>_frames_r02*.json): measured seconds per frame, cited by file
    import glob
    npf_ref = None
    long_runs = {}
    pat = "c4*" if args.config.startswith("c4") else args.config  # the C4 starts share the scene
    for rf in sorted(glob.glob(os.path.join(ROOT, "profiles", f"{pat}_frames_r02*.json"))):
        with open(rf) as f:
            lr = json.load(f)
        tag = os.path.basename(rf)[:-5]
        long_runs[tag] = {k: lr.get(k) for k in ("seconds_per_frame", "newton_per_frame", "frames_converged",
                                                 "frames", "chi", "max_newton", "when")}
        long_runs[tag]["file"] = os.path.relpath(rf, ROOT)
        if lr.get("frames_converged") and npf_ref is None:
            npf_ref = lr.get("newton_per_frame")
    line = {
        "metric": METRIC, "value": pcg_per_s, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if shared else "weak",
        "vs_baseline": None, "dtype": "f64 (SpMV static blocks stored f32)" if args.fp32_matrix else "f64",
        "data": "synthetic",
        "config": {"workload": wl, "tets": int(len(sc["tets"])), "nodes": int(len(sc["rest_x"])),
                   "step": "one inexact-Newton iteration of Alg. 1 (constraint sets, stencils, assembly, warm "
                           "start, PCG, CCD line search, AL updates); frames continue across steps",
                   "parallelism": (f"partitioned{world} (NCCL halo + allreduce)" if shared else
                                   f"replicas{world}" if world > 1 else "single"),
                   "l2": "inputs larger than L2 (system ~0.5 GB/PCG iteration)"},
        "headline": {"ms_per_newton": ms_newton,
                     "active_constraints": {"avg": float(np.mean(nA_t)) if nA_t else None,
                                            "max": int(max(nA_t)) if nA_t else None,
                                            "paper": "228K avg / 292K max (P:664)"},
                     "seconds_per_frame": (float(np.mean([f[0] for f in new_frames])) / 1000.0) if new_frames else None,
                     "seconds_per_frame_note": "frames completed inside the timed region; whole-frame runs: "
                                               "whole_frame_runs"},
        "pcg_iters_per_s_in_pcg": pcg / (d["ms_pcg"] / 1000.0) if d["ms_pcg"] > 0 else None,
        "pcg_microbench": pcg_micro,
        "newton_iters": newton, "pcg_iters": pcg, "pcg_iters_per_newton": ppn,
        "ms_per_newton": ms_newton,
        "phase_ms_per_newton": {k: d[k] / max(newton, 1) for k in
                                ("ms_collision", "ms_assembly", "ms_pcg", "ms_linesearch")},
        "frames_completed_in_timed_region": len(new_frames),
        "frames_hit_newton_cap": run.unconverged,
        "seconds_per_frame": (float(np.mean([f[0] for f in new_frames])) / 1000.0) if new_frames else None,
        "seconds_per_frame_projection": (ms_newton * npf_ref / 1000.0) if npf_ref else None,
        "newton_per_frame_ref": npf_ref,  # from a converged whole-frame run only (projection = ms/Newton x it)
        "whole_frame_runs": long_runs or None,
        "max_constraints": tot1["max_constraints"],
        "roofline": {"kernel": "k_spmv_ts (BSR3 SpMV in PCG)", "bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "peak_source": peak_src, "mean_launch_us": spmv_us, "launches": d_n,
                     "alg_bytes_per_launch": d_alg / max(d_n, 1), "kernel_min_bytes_per_launch": d_mov / max(d_n, 1),
                     "kernel_min_gbs": moved_gbs},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
