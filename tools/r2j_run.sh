# r2j: RK4 trig modes (0 libm, 1 per-stage fast sincos, 2 angle addition): time + parity + tests
mkdir -p gpurun_out
for m in 0 1 2; do PMX_RK4_MODE=$m timeout 300 python tools/rk4_time.py; done > gpurun_out/rk4_modes.log 2>&1
python - >> gpurun_out/rk4_modes.log 2>&1 <<'PY'
import numpy as np, sys
sys.path.insert(0, "oracle")
import oracle as O
sys.path.insert(0, ".")
from paper_2211_00621_b200 import synth
want = O.rk4(synth.rk4_params(10000), synth.RK4_INIT, 1000, synth.RK4_H).reshape(-1)
for m in "012":
    got = np.load(f"gpurun_out/rk4_out_{m}.npy").reshape(-1)
    rel = np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300))
    print("mode", m, "max_rel_vs_oracle", rel)
PY
cat gpurun_out/rk4_modes.log
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "rk4" 2>&1 | tail -3
