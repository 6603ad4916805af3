"""SpMV / PCG variant timing on the bench workload (contact-rich C4 start, first Newton system):
plain product (bal_bench_spmv), 1,000-iteration PCG microbenchmark and the in-PCG SpMV launch time
from the library's CUDA events.  Build variants are selected with BAL_LIB_PATH, runtime switches
with their environment variables; one JSON line per run.
    python tools/spmv_variants.py [c4|c4-drop]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_00046_b200 as bal  # noqa: E402
import scenes  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
sc = scenes.make_puffer_net(seed=4, settled=(cfg == "c4"))
dev = torch.device("cuda:0")
prm = dict(sc["params"])
prm["max_pcg"] = 200
ctx = bal.bal_init(sc, params=prm, flags=int(os.environ.get("BAL_FLAGS", "0")))
x = torch.as_tensor(sc["x0"].ravel(), device=dev)
v = torch.as_tensor(sc["v0"].ravel(), device=dev)
bal.bal_frame_begin(ctx, x, v)
bal.bal_frame_iterate(ctx, 1)
nA = bal.bal_get_trace(ctx, max_records=8)[-1]["nA"]
plain = bal.bal_bench_spmv(ctx, 50)
b = torch.randn(x.numel(), dtype=torch.float64, device=dev)
xo = torch.empty_like(b)
z0 = torch.zeros_like(b)
bal.bal_pcg(ctx, b, z0, xo, warm_start=0, rel_tol=0.0, stall_window=0, max_iters=50)
c0 = bal.bal_spmv_counters(ctx)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
s = bal.bal_pcg(ctx, b, z0, xo, warm_start=0, rel_tol=0.0, stall_window=0, max_iters=1000)
e1.record()
torch.cuda.synchronize()
c1 = bal.bal_spmv_counters(ctx)
n = max(c1["launches"] - c0["launches"], 1)
print(json.dumps({"lib": os.path.basename(bal.lib_path), "env": {k: v for k, v in os.environ.items()
                                                                 if k.startswith("BAL_")},
                  "cfg": cfg, "nA": nA, "plain_spmv_us": plain,
                  "pcg_it_s": 1000.0 * s["iters"] / e0.elapsed_time(e1),
                  "pcg_spmv_us": 1000.0 * (c1["ms"] - c0["ms"]) / n,
                  "alg_MB": (c1["bytes_alg"] - c0["bytes_alg"]) / n / 1e6,
                  "moved_MB": (c1["bytes_moved"] - c0["bytes_moved"]) / n / 1e6}))
