import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import scenes, paper_2407_00046_b200 as bal
from oracle.bal import Oracle
sc = scenes.make_single_tet(1, height=0.01, speed=1.0)
o = Oracle(sc); ctx = bal.bal_init(sc); dev = torch.device("cuda:0")
x = torch.as_tensor(sc["x0"].ravel(), device=dev); v = torch.as_tensor(sc["v0"].ravel(), device=dev)
xn = torch.empty_like(x); vn = torch.empty_like(v)
bal.bal_step(ctx, x, v, xn, vn); tg = bal.bal_get_trace(ctx)
tr = []; o.step(sc["x0"], sc["v0"], tr)
for l in range(max(len(tg), len(tr))):
    a = tg[l] if l < len(tg) else {}; b = tr[l] if l < len(tr) else {}
    print(l, "GPU", {k: round(a.get(k, -1), 6) for k in ("nA", "dmin", "sigma", "pcg_iters", "alpha_ccd", "alpha", "rel_e")})
    print(l, "ORA", {k: (round(float(b.get(k, -1)), 6)) for k in ("nA", "dmin", "sigma", "pcg_iters", "alpha_ccd", "alpha", "rel_e")})
