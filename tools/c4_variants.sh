#!/bin/bash
# C4 variants: Newton convergence of frame 0 under different scene knobs (each capped in wall time)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
run() { name=$1; kw=$2; lim=$3
  BAL_VERBOSE=1 timeout $lim python tools/probe_c4.py 2 "$kw" 2>&1 | grep -v "^\[bal\]  \|bal-ws\|bal-pcg" > gpurun_out/var_$name.log; echo "rc=$?" >> gpurun_out/var_$name.log; }
run chi0 '{"chi": 0.0}' 240
run enet7 '{"E_net": 1e7}' 240
run noballs '{"n_balls": 0}' 240
run nonet_small '{"nx": 3, "nz": 3}' 240
run gap '{"drop_gap": 0.002, "chi": 0.0, "E_net": 1e7}' 240
