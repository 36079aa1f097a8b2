"""Time the RK4 sweep (BASELINE configs[0]: 10^4 parameter sets x 10^3 steps)
with the current kernel; print ms and a checksum.  Run twice with
PMX_RK4_MODE=0|1 to A/B the trig modes (csrc/rk4.cu)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_00621_b200 import rk4_sweep, synth  # noqa: E402

n, m = 10000, 1000
ps = torch.tensor(synth.rk4_params(n), dtype=torch.float64, device="cuda")
s0 = torch.tensor(synth.RK4_INIT, dtype=torch.float64, device="cuda")
for _ in range(3):
    out = rk4_sweep(ps, s0, m, synth.RK4_H)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(10):
    a.record()
    out = rk4_sweep(ps, s0, m, synth.RK4_H)
    b.record()
    b.synchronize()
    ts.append(a.elapsed_time(b))
res = out.data.cpu().numpy()
tag = os.environ.get("PMX_RK4_MODE", "2")
np.save(f"gpurun_out/rk4_out_{tag}.npy", res)
print(json.dumps({"mode": tag, "ms_min": min(ts), "ms_med": sorted(ts)[5]}))
