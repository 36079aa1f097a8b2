"""Diagnostic: max relative log-likelihood error of the HMM forward kernels
against the fp64 log-space oracle (SIMT vs tensor-core path).

    PMX_HMM_SIMT=1 python tools/hmm_precision.py 1024 300 35
"""
import os
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import oracle as O  # noqa: E402
import paper_2211_00621_b200 as P  # noqa: E402
from paper_2211_00621_b200 import synth  # noqa: E402

S, T, NS = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (1024, 300, 35)))
A, E, pi = synth.hmm_model(S, 8)
obs = synth.hmm_obs(NS, T, 8)
got = P.accelerate(P.hmm_forward, A, E, pi, obs)
want = O.hmm_forward(A, E, pi, obs)
rel = (got - want) / np.abs(want)
print(f"S={S} T={T} nsig={NS} simt={os.environ.get('PMX_HMM_SIMT', '0')} "
      f"max_rel={np.max(np.abs(rel)):.3e} mean_rel={np.mean(rel):+.3e} ll0={want[0]:.6f}")
