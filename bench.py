#!/usr/bin/env python
"""Benchmark of the BAL inexact Newton-PCG time step (arXiv 2407.00046) on B200.

Metric (BASELINE.json): "seconds/frame & PCG iters/s at 1.76M tets; BSR SpMV HBM GB/s vs peak".
One bench step = one bal_step = one frame (h = 1/30 s) of the C4 puffer-balls-on-chain-net scene
(configs[3], ~1.7M tets) -- every row of SURVEY §8(a): constraint sets, elastic / contact / friction
stencils, atomic-free assembly, warm start, PCG, CCD line search, AL updates.
`value` = frames/s of the whole job (N ranks each advance their own replica of the scene: weak
scaling, no data-path collective).  Extra keys: seconds/frame, PCG iterations/s, SpMV roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c4|c1]
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
# Newton / PCG counts of the C4 frames observed on the GPU path (profiles/bench_r01.md); used only
# to scale the reference (oracle) arm's bounded sample to a frame.
C4_NEWTON_PER_FRAME = 40.0
C4_PCG_PER_NEWTON = 150.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=["c4", "c1"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def make_scene(cfg):
    import scenes
    if cfg == "c1":
        return scenes.make_cubes(1), "C1 two stacked soft cubes (1.5K tets), dt=1/30 s"
    return scenes.make_puffer_net(seed=4), "C4 puffer balls on chain-net (~1.7M tets), dt=1/30 s"


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


def job_throughput(local_seconds, units_per_rank, world, device):
    """Max of the ranks' timed-region seconds (the job time) and the whole-job throughput
    (units processed by all ranks / job time).  One all_reduce(MAX) when world > 1."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(local_seconds)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    s = float(t.item())
    return s, world * units_per_rank / s


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
                     "mu": m.mu[sel], "lam": m.lam[sel]})
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
    vals = []
    t_all = time.perf_counter()
    info = {}
    for _ in range(max(args.warmup, 0)):
        oracle_sample(sc, C4_NEWTON_PER_FRAME, C4_PCG_PER_NEWTON, budget_tets=2000)
    for k in range(args.steps):
        s_frame, threads, desc, info = oracle_sample(sc, C4_NEWTON_PER_FRAME, C4_PCG_PER_NEWTON, seed=k)
        vals.append(s_frame)
    s_frame = float(np.mean(vals))
    fps = 1.0 / s_frame
    line = {"impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * s_frame, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl, "tets": int(len(sc["tets"])), "nodes": int(len(sc["rest_x"]))},
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": threads, "kind": "oracle", "sample": desc},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "detail": {**info, "wall_s": time.perf_counter() - t_all}}
    print(json.dumps(line), flush=True)


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
    ctx = bal.bal_init(sc, device=local)
    x = torch.as_tensor(sc["x0"].ravel(), device=dev)
    v = torch.as_tensor(sc["v0"].ravel(), device=dev)
    xn, vn = torch.empty_like(x), torch.empty_like(v)
    stream = torch.cuda.current_stream(dev)
    bal.bal_set_stream(ctx, stream)
    for _ in range(args.warmup):
        bal.bal_step(ctx, x, v, xn, vn)
        x, xn = xn, x
        v, vn = vn, v
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    spmv0 = bal.bal_spmv_counters(ctx)
    launches0 = ctx.kernel_launches
    stats = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            stats.append(bal.bal_step(ctx, x, v, xn, vn))
            x, xn = xn, x
            v, vn = vn, v
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = e0.elapsed_time(e1)
    launches = ctx.kernel_launches - launches0
    spmv1 = bal.bal_spmv_counters(ctx)
    s_max, fps = job_throughput(ms / 1000.0, args.steps, world, dev)
    ms_max = 1000.0 * s_max
    s_frame = s_max / args.steps
    pcg = sum(s["pcg_iters"] for s in stats)
    pcg_ms = sum(s["ms_pcg"] for s in stats)
    newton = sum(s["newton_iters"] for s in stats)
    # SpMV roofline from the library's CUDA events around every SpMV launch in the timed region
    d_ms = spmv1["ms"] - spmv0["ms"]
    d_n = spmv1["launches"] - spmv0["launches"]
    d_alg = spmv1["bytes_alg"] - spmv0["bytes_alg"]
    d_mov = spmv1["bytes_moved"] - spmv0["bytes_moved"]
    peak, peak_src = measured_peaks()
    spmv_us = 1000.0 * d_ms / max(d_n, 1)
    achieved = (d_alg / max(d_n, 1)) / (spmv_us * 1e-6) / 1e9 if d_n else None
    moved_gbs = (d_mov / max(d_n, 1)) / (spmv_us * 1e-6) / 1e9 if d_n else None
    traffic = None
    tf = os.path.join(ROOT, "profiles", "spmv_traffic.json")
    if os.path.exists(tf):
        with open(tf) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    # e2e through the public API with host buffers (bal_step_host: H2D + D2H inside the call)
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().numpy()
        vh = v.cpu().numpy()
        ne = max(1, min(args.steps, 2))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(ne):
            xh, vh, _s = bal.bal_step_host(ctx, xh, vh)
        el = time.perf_counter() - t0
        _s, e2e_fps = job_throughput(el, ne, world, dev)
        nb = 2 * 3 * 8 * len(sc["rest_x"])
        e2e = {"value": e2e_fps, "unit": "frames/s", "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb}
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        npf = newton / max(args.steps, 1)
        ppn = pcg / max(newton, 1)
        s_or, threads, desc, _info = oracle_sample(sc, npf, ppn)
        cpu = {"value": 1.0 / s_or, "unit": "frames/s", "cores": threads, "kind": "oracle", "sample": desc}
    line = {
        "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl, "tets": int(len(sc["tets"])), "nodes": int(len(sc["rest_x"])),
                   "parallelism": f"replicas{world}" if world > 1 else "single",
                   "l2": "inputs larger than L2 (system ~0.8 GB/iteration)"},
        "seconds_per_frame": s_frame,
        "pcg_iters_per_s": pcg / (pcg_ms / 1000.0) if pcg_ms > 0 else None,
        "newton_iters_per_frame": newton / args.steps,
        "pcg_iters_per_newton": pcg / max(newton, 1),
        "phase_ms_per_frame": {k: sum(s[k] for s in stats) / args.steps for k in
                               ("ms_collision", "ms_assembly", "ms_pcg", "ms_linesearch", "ms_total")},
        "max_constraints": max(s["max_constraints"] for s in stats),
        "roofline": {"kernel": "k_spmv (BSR3 SpMV in PCG)", "bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "peak_source": peak_src, "mean_launch_us": spmv_us, "launches": d_n,
                     "alg_bytes_per_launch": d_alg / max(d_n, 1), "full_bsr_bytes_per_launch": d_mov / max(d_n, 1),
                     "full_bsr_gbs": moved_gbs},
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
