# r2p: k-mer HMM on CTA pairs with alpha in registers: parity tests, sanitizer, step time vs the global-alpha kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "kmer" > gpurun_out/pytest_kmer.log 2>&1
tail -3 gpurun_out/pytest_kmer.log
timeout 300 compute-sanitizer --tool memcheck python -c "
import numpy as np, sys; sys.path.insert(0,'.')
from paper_2211_00621_b200 import accelerate, hmm_kmer_forward, synth
E = synth.kmer_emission(8, 8); obs = synth.hmm_obs(5, 4, 8)
print(accelerate(lambda em, o: hmm_kmer_forward(8, 0.5, 0.125, em, o), E, obs))" > gpurun_out/kmer_memcheck.log 2>&1
tail -4 gpurun_out/kmer_memcheck.log
timeout 300 compute-sanitizer --tool synccheck python -c "
import numpy as np, sys; sys.path.insert(0,'.')
from paper_2211_00621_b200 import accelerate, hmm_kmer_forward, synth
E = synth.kmer_emission(8, 8); obs = synth.hmm_obs(5, 4, 8)
print(accelerate(lambda em, o: hmm_kmer_forward(8, 0.5, 0.125, em, o), E, obs))" > gpurun_out/kmer_synccheck.log 2>&1
tail -4 gpurun_out/kmer_synccheck.log
(timeout 300 python tools/kmer_time.py 300; PMX_KMER_VEC=1 timeout 300 python tools/kmer_time.py 300; timeout 300 python tools/kmer_time.py 1000) > gpurun_out/kmer_time.log 2>&1
cat gpurun_out/kmer_time.log
