"""NEXT-1 on the bench workload: the first Newton iterations of the contact-rich C4 frame 0 with
block-Jacobi (+ warm start, the paper's method), the App. A additive preconditioner alone, and the
additive preconditioner + warm start; per Newton iteration the global PCG iterations and stop reason,
per variant the PCG milliseconds.  One JSON line per variant.
    python tools/probe_as_c4.py [newton_iters]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_00046_b200 as bal  # noqa: E402
import scenes  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sc = scenes.make_puffer_net(seed=4, settled=True)
dev = torch.device("cuda:0")
for name, fl in (("block-Jacobi + warm start", 0), ("additive alone", bal.BAL_ADDITIVE_PRECOND | bal.BAL_NO_WARMSTART),
                 ("additive + warm start", bal.BAL_ADDITIVE_PRECOND)):
    ctx = bal.bal_init(sc, flags=fl)
    x = torch.as_tensor(sc["x0"].ravel(), device=dev)
    v = torch.as_tensor(sc["v0"].ravel(), device=dev)
    bal.bal_frame_begin(ctx, x, v)
    bal.bal_frame_iterate(ctx, K)
    tr = bal.bal_get_trace(ctx, max_records=K)
    st = bal.bal_frame_stats(ctx)
    print(json.dumps({"variant": name, "pcg_iters": [int(t["pcg_iters"]) for t in tr],
                      "pcg_stop": [int(t["pcg_stop"]) for t in tr], "rel_e": [t["rel_e"] for t in tr],
                      "ms_pcg": st.get("ms_pcg"), "ms_total": st.get("ms_total")}), flush=True)
    del ctx
    torch.cuda.empty_cache()
