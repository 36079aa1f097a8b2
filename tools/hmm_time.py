"""Time the HMM forward kernel at S=1024 (4096 signals) for a given T (ms per
10^4 steps extrapolated).  Env PMX_HMM_TC / PMX_HMM_DBG select variants."""
import os, sys, pathlib
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np, torch
from paper_2211_00621_b200 import _lib, casestudies as CS, synth
T = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
S, K = 1024, 8
nsig = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
A, E, pi = synth.hmm_model(S, K)
dev = torch.device("cuda")
Ad = torch.from_numpy(A.astype(np.float32)).to(dev)
lE = torch.from_numpy(np.log(E).astype(np.float32)).to(dev)
lpi = torch.from_numpy(np.log(pi).astype(np.float32)).to(dev)
obs = torch.from_numpy(synth.hmm_obs(nsig, T, K)).to(dev)
out = torch.empty(nsig, dtype=torch.float64, device=dev)
ws = torch.empty(_lib.load().pmx_hmm_forward_workspace_bytes(S, nsig), dtype=torch.uint8, device=dev)
f = lambda: CS.hmm_forward_raw(lpi, Ad, lE, obs, S, K, nsig, T, out, ws)
f(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); f(); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"tc={os.environ.get('PMX_HMM_TC','f16')} dbg={os.environ.get('PMX_HMM_DBG','0')} nsig={nsig} T={T}: {ms:.2f} ms "
      f"-> {ms * 9999 / (T - 1):.1f} ms at T=10^4, {ms / (T - 1) * 1e3:.2f} us/step")
