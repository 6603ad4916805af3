"""Residual histories of PCG on the C4 first Newton system (cold / warm start, no stagnation stop)."""
import sys, os
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
b = -out["grad"]
bn = b.norm().item()
xo = torch.empty_like(b)
for ws in (0, 1):
    s = bal.bal_pcg(ctx, b, None, xo, warm_start=ws, stall_window=0, max_iters=5000)
    h = bal.bal_pcg_history(ctx) / bn
    ks = [0, 1, 2, 5, 10, 20, 50, 100, 150, 200, 300, 500, 800, 1000, 1500, 2000, 3000, len(h) - 1]
    print("ws", ws, s)
    print("  ", " ".join(f"{k}:{h[k]:.2e}" for k in ks if k < len(h)))
    # windowed minima
    W = 100
    for k in range(W, min(len(h), 1200), W):
        print(f"   k={k} min_recent={h[k-W+1:k+1].min():.3e} min_older={h[:k-W+1].min():.3e} r_k/r_k-W={h[k]/h[k-W]:.3e}")
np.save("gpurun_out/hist_ws.npy", h)
