import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import scenes, paper_2407_00046_b200 as bal
sc = scenes.make_single_tet(1, height=0.01, speed=1.0)
dev = torch.device("cuda:0")
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    ctx = bal.bal_init(sc)
    if trial % 2 == 0:
        xh, vh, s = bal.bal_step_host(ctx, sc["x0"], sc["v0"])
    else:
        x = torch.as_tensor(sc["x0"].ravel(), device=dev); v = torch.as_tensor(sc["v0"].ravel(), device=dev)
        xn = torch.empty_like(x); vn = torch.empty_like(v)
        try:
            s = bal.bal_step(ctx, x, v, xn, vn)
        except bal.BalError as e:
            print("ERR", e); s = None
    tr = bal.bal_get_trace(ctx)
    print(trial, s and s["newton_iters"], len(tr), [ (round(r["alpha_ccd"],4), round(r["alpha"],4), r["nA"], r["pcg_iters"]) for r in tr[:12]])
