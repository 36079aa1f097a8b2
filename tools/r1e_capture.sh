#!/bin/bash
# r1e evidence: ncu --set full of the kernels changed since r1d (RK4 branch-free
# trig, NN bulk-copy/4x4 tiles/warp softmax, ordered reduce coalescing) and a
# launch list of the default bench. Outputs under gpurun_out/.
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rk4 -c 1 \
  -o gpurun_out/prof_rk4 python tools/profile_cases.py rk4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_nn_grad -s 1 -c 1 \
  -o gpurun_out/prof_nn python tools/nn_case.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_reduce_ordered|k_seq_loop_jit" -c 2 \
  -o gpurun_out/prof_generic2 python tools/profile_cases.py generic > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu \
  > gpurun_out/bench_ncu.log 2>&1
ls -la gpurun_out
