"""Mini C4 (3x3 net + one small spiky ball): GPU vs oracle for a couple of steps."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scenes
KW = dict(nx=3, nz=3, n_balls=1, ball_R=5.0, n_spikes=16, spike_len=4.0)
def mini():
    return scenes.make_puffer_net(**KW)
if __name__ == "__main__":
    which = sys.argv[1]
    nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    sc = mini()
    print("T", len(sc["tets"]), "N", len(sc["rest_x"]), flush=True)
    if which == "oracle":
        from oracle.bal import Oracle
        o = Oracle(sc)
        x, v = sc["x0"], sc["v0"]
        for s in range(nsteps):
            tr = []
            t = time.time()
            try:
                x, v, st = o.step(x, v, tr)
            except Exception as e:
                print("ERR", e)
            print("step", s, time.time() - t, len(tr), [round(r["rel_e"], 4) for r in tr][-5:], flush=True)
            for r in tr[:40]:
                print("  ", {k: (float('%.4g' % v_) if isinstance(v_, float) else v_) for k, v_ in r.items() if k not in ("groups", "ws_iters")})
            np.save(f"/tmp/mini_x{s}.npy", x)
    else:
        import torch, paper_2407_00046_b200 as bal
        ctx = bal.bal_init(sc)
        dev = torch.device("cuda:0")
        x = torch.as_tensor(sc["x0"].ravel(), device=dev); v = torch.as_tensor(sc["v0"].ravel(), device=dev)
        for s in range(nsteps):
            xn = torch.empty_like(x); vn = torch.empty_like(v)
            try:
                st = bal.bal_step(ctx, x, v, xn, vn)
            except bal.BalError as e:
                print("ERR", e)
            tr = bal.bal_get_trace(ctx)
            print("step", s, len(tr))
            for r in tr[:40]:
                print("  ", {k: float('%.4g' % v_) for k, v_ in r.items()})
            x, v = xn, vn
