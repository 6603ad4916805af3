"""Long run: whole C4 frames through bal_step (device timing), written to profiles/c4_frames.json.

    python tools/c4_frames.py [n_frames] [--chi X]

Records per frame: seconds (CUDA events), Newton / PCG / warm-start iterations, max |A|, converged,
per-phase ms.  bench.py reads `newton_per_frame` from it for its labelled s/frame projection."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_00046_b200 as bal  # noqa: E402
import scenes  # noqa: E402


def main():
    nf = int(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else 1
    kw = {}
    if "--chi" in sys.argv:
        kw["chi"] = float(sys.argv[sys.argv.index("--chi") + 1])
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else os.path.join("profiles", "c4_frames.json")
    scene = sys.argv[sys.argv.index("--scene") + 1] if "--scene" in sys.argv else "c4"
    make = {"c4": lambda: scenes.make_puffer_net(seed=4, **kw),
            "c4s": lambda: scenes.make_puffer_net(seed=4, settled=True, **kw),
            "c2": lambda: scenes.make_armadillo_like(2, **kw),
            "c3": lambda: scenes.make_impact(3, **kw), "c1": lambda: scenes.make_cubes(1)}[scene]
    sc = make()
    if "--max-newton" in sys.argv:
        sc["params"]["max_newton"] = int(sys.argv[sys.argv.index("--max-newton") + 1])
    dev = torch.device("cuda:0")
    flags = bal.BAL_FRICTION_LAGGED if "--lagged-friction" in sys.argv else 0
    if "--no-freeze" in sys.argv:
        flags |= bal.BAL_FRICTION_NO_FREEZE
    ctx = bal.bal_init(sc, flags=flags)
    st = torch.cuda.current_stream(dev)
    x = torch.as_tensor(sc["x0"].ravel(), device=dev)
    v = torch.as_tensor(sc["v0"].ravel(), device=dev)
    frames = []
    for f in range(nf):
        xn, vn = torch.empty_like(x), torch.empty_like(v)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        bal.bal_frame_begin(ctx, x, v)
        while not bal.bal_frame_iterate(ctx, 16):
            s = bal.bal_frame_stats(ctx)
            print(f"  frame {f}: newton {s['newton_iters']} pcg {s['pcg_iters']} t {s['ms_total'] / 1e3:.1f}s "
                  f"rel_grad {s['last_rel_grad']:.3e}", flush=True)
            if s["newton_iters"] >= sc["params"]["max_newton"]:
                break
        s = bal.bal_frame_finish(ctx, xn, vn, allow_unconverged=True)
        e1.record(st)
        torch.cuda.synchronize()
        rec = {"frame": f, "seconds": e0.elapsed_time(e1) / 1e3, **{k: (float(v_) if isinstance(v_, float) else v_)
                                                                      for k, v_ in s.items()}}
        frames.append(rec)
        print(json.dumps(rec), flush=True)
        x, v = xn, vn
    conv = [fr for fr in frames if fr["converged"]]
    res = {"scene": sc["name"] + "".join(f", {k}={v}" for k, v in kw.items())
                    + (" with BAL_FRICTION_LAGGED" if flags & bal.BAL_FRICTION_LAGGED else "")
                    + (" with BAL_FRICTION_NO_FREEZE" if flags & bal.BAL_FRICTION_NO_FREEZE else ""),
           "chi": float(sc["params"]["chi"]), "flags": int(flags),
           "tets": int(len(sc["tets"])), "nodes": int(len(sc["rest_x"])),
           "gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "frames": frames,
           "newton_per_frame": float(np.mean([fr["newton_iters"] for fr in (conv or frames)])),
           "seconds_per_frame": float(np.mean([fr["seconds"] for fr in (conv or frames)])),
           "frames_converged": len(conv), "max_newton": int(sc["params"]["max_newton"]),
           "note": "newton_per_frame / seconds_per_frame: mean over the converged frames (over all frames, "
                   "Newton cap included, when none converged)"}
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps({k: v_ for k, v_ in res.items() if k != "frames"}))


if __name__ == "__main__":
    main()
