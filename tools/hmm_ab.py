"""Run the HMM forward kernel selected by PMX_HMM_TC (env; default: the 4-CTA
pair-UMMA kernel) on fixed inputs and save the log-likelihoods to
gpurun_out/hmm_ll_<variant>.npy, so two runs can be compared.
    python tools/hmm_ab.py [nsig] [T]"""
import os, sys, pathlib, subprocess, json
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np, torch
from paper_2211_00621_b200 import _lib, casestudies as CS, synth
nsig = int(sys.argv[1]) if len(sys.argv) > 1 else 256
T = int(sys.argv[2]) if len(sys.argv) > 2 else 50
S, K = 1024, 8
A, E, pi = synth.hmm_model(S, K)
dev = torch.device("cuda")
Ad = torch.from_numpy(A.astype(np.float32)).to(dev)
lE = torch.from_numpy(np.log(E).astype(np.float32)).to(dev)
lpi = torch.from_numpy(np.log(pi).astype(np.float32)).to(dev)
obs = torch.from_numpy(synth.hmm_obs(nsig, T, K)).to(dev)
out = torch.empty(nsig, dtype=torch.float64, device=dev)
ws = torch.empty(_lib.load().pmx_hmm_forward_workspace_bytes(S, nsig), dtype=torch.uint8, device=dev)
CS.hmm_forward_raw(lpi, Ad, lE, obs, S, K, nsig, T, out, ws)
torch.cuda.synchronize()
np.save(f"gpurun_out/hmm_ll_{os.environ.get('PMX_HMM_TC', 'default')}.npy", out.cpu().numpy())
print(os.environ.get("PMX_HMM_TC", "default"), out[:4].tolist())
