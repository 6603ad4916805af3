"""NEXT-1 ablations on the same kernels: warm start on/off (Fig. warm
start), BAL vs plain inexact-Newton IPC (A' = empty, sigma = sigma^0), the capped and the
min readings of the sigma schedule (Alg. 1 line 16), the two-level additive preconditioner of
App. A alone and with the warm start.  Runs whole frames of a scene through
bal_frame_* with each flag set and prints per-variant totals as JSON lines.

    python tools/ablation.py c1|c2|c3 [frames]      # whole frames
    python tools/ablation.py c4 [newton_iters]      # C4 drop start: the first K Newton iterations of frame 0
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_00046_b200 as bal  # noqa: E402
import scenes  # noqa: E402

VARIANTS = {"bal+warmstart": 0, "bal, no warm start": bal.BAL_NO_WARMSTART,
            "inexact Newton (no AL)": bal.BAL_NO_AUGLAG, "sigma cap 1e8 sigma0": bal.BAL_SIGMA_CAP,
            "sigma min(1.2 sigma, 100 sigma0)": bal.BAL_SIGMA_MIN,
            "additive precond (App. A) alone": bal.BAL_ADDITIVE_PRECOND | bal.BAL_NO_WARMSTART,
            "additive precond + warm start": bal.BAL_ADDITIVE_PRECOND,
            "fp32 matrix storage (NEXT-3)": bal.BAL_FP32_MATRIX,
            "App. B criterion (i) truncated Newton": bal.BAL_PCG_CRIT_I,
            "App. B criterion (ii) u kappa ||x||": bal.BAL_PCG_CRIT_II,
            "App. B criterion (iii) u kappa ||b||": bal.BAL_PCG_CRIT_III}
ONLY = os.environ.get("BAL_ABL_ONLY")  # comma-separated substrings: run only the matching variants


def run(sc, flags, frames=None, newton=None):
    dev = torch.device("cuda:0")
    ctx = bal.bal_init(sc, flags=flags)
    st = torch.cuda.current_stream(dev)
    x = torch.as_tensor(sc["x0"].ravel(), device=dev)
    v = torch.as_tensor(sc["v0"].ravel(), device=dev)
    tot = {"newton_iters": 0, "pcg_iters": 0, "ws_iters": 0, "frames": 0, "converged": 0}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(frames or 1):
        xn, vn = torch.empty_like(x), torch.empty_like(v)
        bal.bal_frame_begin(ctx, x, v)
        if newton:
            bal.bal_frame_iterate(ctx, newton)
        else:
            bal.bal_frame_iterate(ctx, sc["params"]["max_newton"])
        s = bal.bal_frame_finish(ctx, xn, vn, allow_unconverged=True)
        for k in ("newton_iters", "pcg_iters", "ws_iters"):
            tot[k] += s[k]
        tot["frames"] += 1
        tot["converged"] += int(s["converged"])
        x, v = xn, vn
    e1.record(st)
    torch.cuda.synchronize()
    tot["seconds"] = e0.elapsed_time(e1) / 1e3
    return tot


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "c1"
    k = int(sys.argv[2]) if len(sys.argv) > 2 else (10 if which == "c1" else 20)
    sc = {"c1": lambda: scenes.make_cubes(1), "c2": lambda: scenes.make_armadillo_like(2),
          "c3": lambda: scenes.make_impact(3), "c4": lambda: scenes.make_puffer_net(seed=4)}[which]()
    for name, fl in VARIANTS.items():
        if ONLY and not any(k in name for k in ONLY.split(",")):
            continue
        try:
            r = run(sc, fl, newton=k) if which == "c4" else run(sc, fl, frames=k)
        except bal.BalError as e:  # a variant that fails (e.g. NaN) is reported, not fatal
            r = {"error": str(e)}
        print(json.dumps({"scene": which, "variant": name, **r}), flush=True)


if __name__ == "__main__":
    main()
