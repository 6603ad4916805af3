"""Driver for ncu on the bench workload: the contact-rich C4 start, one inexact-Newton iteration of
frame 0 (the library's own constraint set, ~2.5e5 pairs), then SpMV launches on that system.
    ncu -k regex:k_spmv_ts -c 1 python tools/prof_spmv_settled.py
profiles the first plain product of the Newton iteration (A x0 of the PCG init, same system)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_00046_b200 as bal  # noqa: E402
import scenes  # noqa: E402

sc = scenes.make_puffer_net(seed=4, settled=True)
dev = torch.device("cuda:0")
prm = dict(sc["params"])
prm["max_pcg"] = int(sys.argv[1]) if len(sys.argv) > 1 else 200
ctx = bal.bal_init(sc, params=prm)
x = torch.as_tensor(sc["x0"].ravel(), device=dev)
v = torch.as_tensor(sc["v0"].ravel(), device=dev)
bal.bal_frame_begin(ctx, x, v)
bal.bal_frame_iterate(ctx, 1)
print("constraints", bal.bal_get_trace(ctx, max_records=8)[-1]["nA"])
print("bench spmv us", bal.bal_bench_spmv(ctx, 20))
c = bal.bal_spmv_counters(ctx)
print("alg bytes/launch", c["bytes_alg"] / max(c["launches"], 1), "moved bytes/launch", c["bytes_moved"] / max(c["launches"], 1))
