"""Diagnose the twisting-rods frame that stalls: run frames 0..K-1 with bal_step, then frame K with
the frame API, printing the decision trace every `every` Newton iterations.
    python tools/rods_diag.py [K] [max_newton] [every] [flags]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_00046_b200 as bal  # noqa: E402
import scenes  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 24
MAXN = int(sys.argv[2]) if len(sys.argv) > 2 else 400
EVERY = int(sys.argv[3]) if len(sys.argv) > 3 else 25
FLAGS = int(sys.argv[4]) if len(sys.argv) > 4 else 0
sc = scenes.make_twisting_rods()
dev = torch.device("cuda:0")
ctx = bal.bal_init(sc, flags=FLAGS)
h = sc["params"]["h"]
fixed = sc["node_fixed"].astype(bool)
x = sc["x0"].copy()
v = np.zeros_like(x)
for k in range(K + 1):
    x[fixed] = scenes.twist_targets(sc, (k + 1) * h)[fixed]
    xt = torch.as_tensor(x.ravel(), device=dev)
    vt = torch.as_tensor(v.ravel(), device=dev)
    if k < K:
        xn, vn = torch.empty_like(xt), torch.empty_like(vt)
        s = bal.bal_step(ctx, xt, vt, xn, vn)
        x, v = xn.cpu().numpy().reshape(-1, 3), vn.cpu().numpy().reshape(-1, 3)
        continue
    bal.bal_frame_begin(ctx, xt, vt)
    done = 0
    while done < MAXN:
        conv = bal.bal_frame_iterate(ctx, EVERY)
        done += EVERY
        tr = bal.bal_get_trace(ctx, max_records=100000)
        last = tr[-EVERY:]
        print(json.dumps({"newton": len(tr), "rel_e_last": last[-1]["rel_e"], "rel_e_min": min(t["rel_e"] for t in tr),
                          "nA": last[-1]["nA"], "nAp": last[-1]["nAp"], "sigma": last[-1]["sigma"],
                          "alpha": [round(t["alpha"], 4) for t in last[-6:]],
                          "alpha_ccd": [round(t["alpha_ccd"], 4) for t in last[-6:]],
                          "halvings": [int(t["halvings"]) for t in last[-6:]],
                          "pcg": [int(t["pcg_iters"]) for t in last[-6:]], "stop": [int(t["pcg_stop"]) for t in last[-6:]],
                          "resumes": sum(int(t["resumes"]) for t in last), "safeguard": sum(int(t["safeguard"]) for t in last)}),
              flush=True)
        if conv:
            print("converged at", len(tr))
            break
