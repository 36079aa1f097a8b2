"""seqLoop cost per step: the bench stencil (m = 2^24 fp64) at 1/5/20/40 steps;
the slope is the per-step streaming time, the intercept the call overhead
(state copy, allocation, launch).  r1f: 65 us/step marginal (0.63 of HBM)."""
import sys, torch
sys.path.insert(0, "/root/repo")
import paper_2211_00621_b200 as P
from paper_2211_00621_b200 import _lib
from paper_2211_00621_b200.runtime import DeviceSeq
ms_ = 1 << 24
s_state = DeviceSeq(torch.arange(ms_, dtype=torch.float64, device="cuda") % 97, (ms_,), _lib.PMX_F64)
stencil = P.lam("x", "j", "t", P.mulf(0.5, P.addf("x", P.get(P.PREV, P.modi(P.addi("j", 1), ms_)))))
for steps in (1, 5, 20, 40):
    P.seq_loop(steps, stencil, s_state); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        a.record(); P.seq_loop(steps, stencil, s_state); b.record(); b.synchronize(); best = min(best, a.elapsed_time(b))
    print(steps, round(best, 3), "ms", round(best / steps * 1e3, 1), "us/step")
