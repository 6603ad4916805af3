"""Probe the contact-rich C4 start (scenes.make_puffer_net(settled=True)): feasibility, |A| and the
cost of a few inexact-Newton iterations."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_00046_b200 as bal  # noqa: E402
import scenes  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sc = scenes.make_puffer_net(seed=4, settled=True)
dev = torch.device("cuda:0")
ctx = bal.bal_init(sc)
x = torch.as_tensor(sc["x0"].ravel(), device=dev)
v = torch.as_tensor(sc["v0"].ravel(), device=dev)
t0 = time.time()
bal.bal_frame_begin(ctx, x, v)
print("frame_begin ok", time.time() - t0, flush=True)
for k in range(n):
    t0 = time.time()
    conv = bal.bal_frame_iterate(ctx, 1)
    st = bal.bal_frame_stats(ctx)
    print(k, "conv", conv, "s", round(time.time() - t0, 3), {q: st[q] for q in ("newton_iters", "pcg_iters", "max_constraints", "ms_collision", "ms_assembly", "ms_pcg", "ms_linesearch")}, flush=True)
tr = bal.bal_get_trace(ctx) if hasattr(bal, "bal_get_trace") else None
