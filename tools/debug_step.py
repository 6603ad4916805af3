"""Debug: GPU vs oracle decision traces on C1 (prints side by side)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import scenes
import paper_2407_00046_b200 as bal
from oracle.bal import Oracle

nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sc = scenes.make_cubes(1)
o = Oracle(sc)
ctx = bal.bal_init(sc)
dev = torch.device("cuda:0")
x = torch.as_tensor(sc["x0"].ravel(), device=dev); v = torch.as_tensor(sc["v0"].ravel(), device=dev)
xo, vo = sc["x0"], sc["v0"]
keys = ["nA", "nAp", "rebuilt", "dmin", "sigma", "ws_iters", "pcg_iters", "pcg_stop", "alpha_ccd", "alpha", "halvings", "resumes", "rel_e"]
for s in range(nsteps):
    xn = torch.empty_like(x); vn = torch.empty_like(v)
    err = None
    try:
        st = bal.bal_step(ctx, x, v, xn, vn)
    except bal.BalError as e:
        err = str(e)
    tg = bal.bal_get_trace(ctx)
    tr = []
    xo, vo, _ = o.step(xo, vo, tr)
    print(f"=== step {s} gpu_err={err}")
    for l in range(max(len(tg), len(tr))):
        a = tg[l] if l < len(tg) else {}
        b = tr[l] if l < len(tr) else {}
        print(l, "GPU", " ".join(f"{k}={a.get(k, float('nan')):.4g}" for k in keys))
        bb = {k: (sum(b[k].values()) if isinstance(b.get(k), dict) else b.get(k, float('nan'))) for k in keys}
        bb["ws_iters"] = max(b["ws_iters"].values()) if b.get("ws_iters") else 0
        print(l, "ORA", " ".join(f"{k}={float(bb[k]):.4g}" for k in keys))
    if err:
        break
    x, v = xn, vn
    print("pos rel err", np.linalg.norm(x.cpu().numpy().reshape(-1, 3) - xo) / np.linalg.norm(xo))
