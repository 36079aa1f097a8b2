#!/bin/bash
# Round-1 evidence run on one B200: bench, launch list, ncu --set full of the
# hot kernels. Outputs under gpurun_out/ (summaries are copied to profiles/).
set -x
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-case-studies --no-cpu \
  > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_map_reduce_vec -c 1 \
  -o gpurun_out/prof_mapreduce python tools/profile_cases.py mapreduce > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_map_reduce_vec|k_loop_vec|k_seq_loop_jit|k_reduce_ordered" -c 4 \
  -o gpurun_out/prof_generic python tools/profile_cases.py generic > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hmm_fwd_pair -c 1 \
  -o gpurun_out/prof_hmm python tools/profile_cases.py hmm > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kmer_fwd_vec -c 1 \
  -o gpurun_out/prof_kmer python tools/profile_cases.py kmer > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc -c 1 \
  -o gpurun_out/prof_knn python tools/profile_cases.py knn > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_nn_grad -c 1 \
  -o gpurun_out/prof_nn python tools/nn_case.py > /dev/null 2>&1
ls -la gpurun_out
