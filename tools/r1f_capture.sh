#!/bin/bash
# r1f evidence run on one B200: GPU tests, smoke, bench line, launch list and
# ncu --set full of the HMM quad kernel and the NN kernel. Outputs under gpurun_out/.
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu \
  > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hmm_fwd_quad -c 1 \
  -o gpurun_out/prof_hmm_quad python tools/hmm_time.py 100 > /dev/null 2>&1
ls -la gpurun_out
