"""Probe: C4 scene on the GPU -- init time, per-frame stats and Newton traces."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import scenes, paper_2407_00046_b200 as bal
nframes = int(sys.argv[1]) if len(sys.argv) > 1 else 1
kw = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
t = time.time(); sc = scenes.make_puffer_net(**kw); print("gen", time.time() - t, len(sc["tets"]), len(sc["rest_x"]), flush=True)
dev = torch.device("cuda:0")
t = time.time(); ctx = bal.bal_init(sc); torch.cuda.synchronize(); print("init", time.time() - t, flush=True)
x = torch.as_tensor(sc["x0"].ravel(), device=dev); v = torch.as_tensor(sc["v0"].ravel(), device=dev)
for f in range(nframes):
    xn = torch.empty_like(x); vn = torch.empty_like(v)
    t = time.time()
    try:
        s = bal.bal_step(ctx, x, v, xn, vn)
    except bal.BalError as e:
        print("ERR", e); s = None
    el = time.time() - t
    tr = bal.bal_get_trace(ctx)
    print(f"frame {f}: {el:.2f}s", json.dumps({k: (round(v_, 3) if isinstance(v_, float) else v_) for k, v_ in (s or {}).items()}), flush=True)
    for r in tr[:60]:
        print("  ", " ".join(f"{k}={r[k]:.4g}" for k in ("l", "nA", "nAp", "dmin", "sigma", "ws_iters", "pcg_iters", "pcg_stop", "alpha_ccd", "alpha", "halvings", "resumes", "rel_e")), flush=True)
    if s is None:
        break
    x, v = xn, vn
print("spmv", bal.bal_spmv_counters(ctx))
