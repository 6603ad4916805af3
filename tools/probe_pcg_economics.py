"""PCG economics on the contact-rich C4 start: residual and CG-objective histories of the global
solves of the first Newton iterations; where stagnation thresholds (R-PCG1 with other constants)
would have stopped.  Writes gpurun_out/pcg_econ.json."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_00046_b200 as bal  # noqa: E402
import scenes  # noqa: E402

settled = "--drop" not in sys.argv
sc = scenes.make_puffer_net(seed=4, settled=settled)
dev = torch.device("cuda:0")
ctx = bal.bal_init(sc)
x = torch.as_tensor(sc["x0"].ravel(), device=dev)
v = torch.as_tensor(sc["v0"].ravel(), device=dev)
bal.bal_frame_begin(ctx, x, v)
res = []
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 3):
    bal.bal_frame_iterate(ctx, 1)
    r = bal.bal_pcg_history(ctx)
    d = bal.bal_pcg_objective_history(ctx)
    tr = bal.bal_get_trace(ctx, max_records=64)[-1]
    stops = {}
    for tau in (1e-2, 1e-3, 1e-4, 1e-6, 1e-8, 1e-10):
        k = next((k for k in range(100, len(d)) if d[k] - d[k - 100] <= tau * d[k]), None)
        stops[str(tau)] = None if k is None else {"k": k, "rel_res": float(r[k] / r[0]), "dec_frac": float(d[k] / d[-1])}
    rec = {"newton": it, "nA": tr["nA"], "pcg_iters": len(r) - 1, "stop": tr["pcg_stop"], "rel_e": tr["rel_e"],
           "alpha": tr["alpha"], "r0": float(r[0]), "r_min_rel": float(r.min() / r[0]), "r_end_rel": float(r[-1] / r[0]),
           "r_every_500": (r[::500] / r[0]).tolist(), "dec_every_500": (d[::500] / max(d[-1], 1e-300)).tolist(),
           "stagnation_stops": stops}
    res.append(rec)
    print(json.dumps({k: rec[k] for k in ("newton", "nA", "pcg_iters", "stop", "rel_e", "alpha", "r_min_rel", "r_end_rel")}),
          json.dumps(stops), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
with open(os.path.join("gpurun_out", "pcg_econ%s.json" % ("" if settled else "_drop")), "w") as f:
    json.dump(res, f, indent=1)
