"""Probe PCG convergence on the C4 first Newton system (no contacts at t=0)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import scenes, paper_2407_00046_b200 as bal
sc = scenes.make_puffer_net()
p = sc["params"]
dev = torch.device("cuda:0")
ctx = bal.bal_init(sc)
x = torch.as_tensor(sc["x0"].ravel(), device=dev)
y = sc["x0"] + p["h"] * sc["v0"] + p["h"] ** 2 * np.array(p["gravity"])[None]
y[sc["node_fixed"] == 1] = sc["x0"][sc["node_fixed"] == 1]
out = bal.bal_assemble(ctx, x, y=y)
g = out["grad"]
b = -g
print("|g|", g.norm().item(), "groups", np.unique(out["group"].cpu().numpy(), return_counts=True))
xo = torch.empty_like(b)
for ws, win, mx in [(1, 100, 20000), (0, 100, 20000), (1, 0, 20000), (0, 0, 20000), (1, 1000, 20000)]:
    torch.cuda.synchronize(); t = time.time()
    s = bal.bal_pcg(ctx, b, None, xo, warm_start=ws, stall_window=win, max_iters=mx)
    torch.cuda.synchronize(); el = time.time() - t
    print(f"ws={ws} window={win}: {s}  {el:.3f}s  {1000*el/max(s['iters'],1):.3f} ms/it", flush=True)
print("spmv", bal.bal_spmv_counters(ctx))
us = bal.bal_bench_spmv(ctx, 50)
print("bench spmv us", us)
