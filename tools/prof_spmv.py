"""Small driver for ncu: C4 first Newton system, a few SpMV + PCG iterations (no stagnation test)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import scenes, paper_2407_00046_b200 as bal
sc = scenes.make_puffer_net(**({"voxel": float(sys.argv[1])} if len(sys.argv) > 1 else {}))
p = sc["params"]
dev = torch.device("cuda:0")
ctx = bal.bal_init(sc)
x = torch.as_tensor(sc["x0"].ravel(), device=dev)
y = sc["x0"] + p["h"] * sc["v0"] + p["h"] ** 2 * np.array(p["gravity"])[None]
y[sc["node_fixed"] == 1] = sc["x0"][sc["node_fixed"] == 1]
out = bal.bal_assemble(ctx, x, y=y)
b = -out["grad"]
xo = torch.empty_like(b)
s = bal.bal_pcg(ctx, b, None, xo, warm_start=0, stall_window=0, max_iters=40)
print(s)
print("bench spmv us", bal.bal_bench_spmv(ctx, 20))
c = bal.bal_spmv_counters(ctx)
print("alg bytes/launch", c["bytes_alg"] / max(c["launches"], 1), "moved bytes/launch", c["bytes_moved"] / max(c["launches"], 1))
