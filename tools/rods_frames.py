"""NEXT-2: whole frames of the twisting-rods scene (Table 1) on one GPU.
Before every step the rod ends (Dirichlet nodes) are moved to their scripted positions at t_{k+1}
(scenes.twist_targets: +-5/12 rev/s about the bundle axis); bal_step then solves the frame with them
fixed (App. C).  One JSON line per frame and a summary; stops at the frame or time limit.
    python tools/rods_frames.py [frames] [seconds] [out.json]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_00046_b200 as bal  # noqa: E402
import scenes  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 30
LIMIT = float(sys.argv[2]) if len(sys.argv) > 2 else 900.0
OUT = sys.argv[3] if len(sys.argv) > 3 else None
sc = scenes.make_twisting_rods()
dev = torch.device("cuda:0")
ctx = bal.bal_init(sc, flags=int(os.environ.get("BAL_FLAGS", "0")))
h = sc["params"]["h"]
fixed = sc["node_fixed"].astype(bool)
x = sc["x0"].copy()
v = np.zeros_like(x)
frames = []
t_start = time.time()
for k in range(F):
    x[fixed] = scenes.twist_targets(sc, (k + 1) * h)[fixed]
    xt = torch.as_tensor(x.ravel(), device=dev)
    vt = torch.as_tensor(v.ravel(), device=dev)
    xn, vn = torch.empty_like(xt), torch.empty_like(vt)
    t0 = time.time()
    try:
        s = bal.bal_step(ctx, xt, vt, xn, vn)
    except bal.BalError as e:
        frames.append({"frame": k, "error": str(e)})
        print(json.dumps(frames[-1]), flush=True)
        break
    torch.cuda.synchronize()
    rec = {"frame": k, "seconds": time.time() - t0, "newton_iters": s["newton_iters"], "pcg_iters": s["pcg_iters"],
           "max_constraints": s["max_constraints"], "min_distance": s["min_distance"]}
    frames.append(rec)
    print(json.dumps(rec), flush=True)
    x = xn.cpu().numpy().reshape(-1, 3)
    v = vn.cpu().numpy().reshape(-1, 3)
    if time.time() - t_start > LIMIT:
        break
ok = [f for f in frames if "error" not in f]
summ = {"scene": "twisting-rods", "flags": int(os.environ.get("BAL_FLAGS", "0")), "tets": len(sc["tets"]), "nodes": len(sc["x0"]), "frames": len(ok),
        "seconds_per_frame": float(np.mean([f["seconds"] for f in ok[1:]])) if len(ok) > 1 else None,
        "newton_per_frame": float(np.mean([f["newton_iters"] for f in ok])) if ok else None,
        "max_constraints": max([f["max_constraints"] for f in ok], default=0),
        "paper": "Table 1 (RTX 4090): 24.1 Newton / frame, 15.54 s / frame, 617K avg / 5.7M max constraints over 18 rounds"}
print(json.dumps(summ), flush=True)
if OUT:
    with open(OUT, "w") as f:
        json.dump({"summary": summ, "frames": frames}, f, indent=1)
