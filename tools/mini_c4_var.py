"""Mini C4 variants on the GPU: Newton iteration counts per step for chi / warm-start / AL ablations."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import scenes, paper_2407_00046_b200 as bal
from tools.mini_c4 import KW
dev = torch.device("cuda:0")
for name, kw, flags in [("chi0", dict(chi=0.0), 0), ("chi0.3", dict(chi=0.3), 0), ("chi0_nows", dict(chi=0.0), 1),
                        ("chi0.3_nows", dict(chi=0.3), 1)]:
    sc = scenes.make_puffer_net(**{**KW, **kw})
    ctx = bal.bal_init(sc, flags=flags)
    x = torch.as_tensor(sc["x0"].ravel(), device=dev); v = torch.as_tensor(sc["v0"].ravel(), device=dev)
    res = []
    for s in range(4):
        xn = torch.empty_like(x); vn = torch.empty_like(v)
        try:
            st = bal.bal_step(ctx, x, v, xn, vn)
            res.append((st["newton_iters"], int(st["pcg_iters"]), round(st["ms_total"])))
        except bal.BalError as e:
            res.append(("ERR", str(e)[:120])); break
        x, v = xn, vn
    print(name, res, flush=True)
