"""Time the k-mer HMM forward (S = 65536, 1024 signals) at a given T; prints ms
and the first log-likelihoods (compare runs of two kernel versions)."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2211_00621_b200 import _lib, synth
T = int(sys.argv[1]) if len(sys.argv) > 1 else 300
km, K, nsig = 8, 8, 1024
lE = torch.from_numpy(np.log(synth.kmer_emission(km, K)).astype(np.float32)).cuda()
obs = torch.from_numpy(synth.hmm_obs(nsig, T, K)).cuda()
out = torch.empty(nsig, dtype=torch.float64, device="cuda")
lib = _lib.load()
ws = torch.empty(lib.pmx_hmm_kmer_workspace_bytes(km, nsig), dtype=torch.uint8, device="cuda")
run = lambda: _lib.check(lib.pmx_hmm_kmer_forward_f32(km, 0.5, 0.125, lE.data_ptr(), K, obs.data_ptr(), nsig, T,
                                                       out.data_ptr(), ws.data_ptr(), ws.numel(),
                                                       torch.cuda.current_stream().cuda_stream), "kmer")
run(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); run(); b.record(); b.synchronize()
ms = a.elapsed_time(b)
print(f"T={T}: {ms:.2f} ms -> {ms * 5999 / (T - 1):.1f} ms at T=6000; ll[:3] = {out[:3].tolist()}")
