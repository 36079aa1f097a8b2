import time, sys, cProfile, pstats
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2211_00621_b200 as P
from paper_2211_00621_b200 import synth
n, m = 10000, 1000
ps = synth.rk4_params(n)
s0 = np.array(synth.RK4_INIT)
pps = torch.from_numpy(ps).pin_memory()
for _ in range(5):
    P.accelerate(lambda p, s: P.rk4_sweep(p, s, m, synth.RK4_H), pps, s0)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(50):
    P.accelerate(lambda p, s: P.rk4_sweep(p, s, m, synth.RK4_H), pps, s0)
torch.cuda.synchronize()
print("accelerate ms", (time.perf_counter() - t) / 50 * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(50):
    P.accelerate(lambda p, s: P.rk4_sweep(p, s, m, synth.RK4_H), pps, s0)
pr.disable()
pstats.Stats(pr).sort_stats('cumulative').print_stats(25)
