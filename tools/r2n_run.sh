# r2n: HMM forward with the per-signal sums moved after the u_t stores: parity tests + step time
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "hmm_forward" > gpurun_out/pytest_hmm.log 2>&1
tail -3 gpurun_out/pytest_hmm.log
timeout 300 python tools/hmm_time.py 1000 4096 > gpurun_out/hmm_time.log 2>&1; cat gpurun_out/hmm_time.log
