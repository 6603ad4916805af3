"""C4 variants: per-frame Newton/PCG counts and time.  argv: nframes, scene-kwargs JSON, params JSON."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import scenes, paper_2407_00046_b200 as bal
nframes = int(sys.argv[1]); kw = json.loads(sys.argv[2]); pp = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {}
sc = scenes.make_puffer_net(**kw); sc["params"].update(pp)
dev = torch.device("cuda:0")
ctx = bal.bal_init(sc, flags=int(pp.get("flags", 0)))
x = torch.as_tensor(sc["x0"].ravel(), device=dev); v = torch.as_tensor(sc["v0"].ravel(), device=dev)
print(kw, pp, len(sc["tets"]), flush=True)
for f in range(nframes):
    xn = torch.empty_like(x); vn = torch.empty_like(v)
    t = time.time()
    try:
        s = bal.bal_step(ctx, x, v, xn, vn); err = ""
    except bal.BalError as e:
        s = {}; err = str(e)[:90]
    tr = bal.bal_get_trace(ctx)
    print(f"  frame {f}: {time.time()-t:.1f}s newton={len(tr)} pcg={sum(r['pcg_iters'] for r in tr):.0f} "
          f"maxA={max([r['nA'] for r in tr] or [0]):.0f} last_rel_e={tr[-1]['rel_e'] if tr else -1:.2e} {err}", flush=True)
    x, v = xn, vn
c = bal.bal_spmv_counters(ctx)
print("  spmv us/launch", 1000 * c["ms"] / max(c["launches"], 1), "alg GB/s", c["bytes_alg"] / max(c["ms"], 1e-9) / 1e6,
      "moved GB/s", c["bytes_moved"] / max(c["ms"], 1e-9) / 1e6, flush=True)
