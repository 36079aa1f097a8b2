"""Time the k-NN kernels at the BASELINE config (2^20 train x 2^16 queries,
d = 64, k = 8) through pmx_knn_f32 with device-resident inputs; print the
median ms.  (The r1 PMX_KNN_PROBE pipeline-only variants were removed from
the kernel; the variable is only echoed for old logs.)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_00621_b200 import _lib, casestudies as CS, synth  # noqa: E402

ntr, nq, d, k, c = 1 << 20, 1 << 16, 64, 8, 10
X = torch.from_numpy(synth.knn_train(ntr, d)).cuda()
Q = torch.from_numpy(synth.knn_query(nq, d)).cuda()
L = torch.from_numpy(synth.knn_labels(ntr, c)).cuda()
out = torch.empty(nq, dtype=torch.int32, device="cuda")
ws = torch.empty(_lib.load().pmx_knn_workspace_bytes(ntr, nq, d, k), dtype=torch.uint8, device="cuda")
for _ in range(60):                       # >= 0.5 s of work: clocks ramped before timing
    CS.knn_raw(X, L, Q, ntr, nq, d, k, c, out, None, ws)
torch.cuda.synchronize()
ts = []
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(7):
    a.record()
    CS.knn_raw(X, L, Q, ntr, nq, d, k, c, out, None, ws)
    b.record()
    b.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
print(f"probe={os.environ.get('PMX_KNN_PROBE', '0')} ms={ts[len(ts) // 2]:.3f} min={ts[0]:.3f}")
