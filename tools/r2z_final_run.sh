# r2z: final evidence refresh of round 2: full GPU tests, smoke, bench (ours +
# reference arm), launch list, ncu --set full of k_knn_tc (full config), k_seq_loop_jit and k_viterbi_pruned
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/r2z_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-parity > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc -c 1 -o gpurun_out/r2z_prof_knn python tools/profile_cases.py knn_full > /dev/null 2>&1
ncu -i gpurun_out/r2z_prof_knn.ncu-rep --page raw --csv > gpurun_out/r2z_knn_raw.csv 2>/dev/null
ncu -i gpurun_out/r2z_prof_knn.ncu-rep --page source --csv > gpurun_out/r2z_knn_source.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_seq_loop_jit -c 1 -o gpurun_out/r2z_prof_seq python tools/profile_cases.py generic > /dev/null 2>&1
ncu -i gpurun_out/r2z_prof_seq.ncu-rep --page raw --csv > gpurun_out/r2z_seq_raw.csv 2>/dev/null
ls gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_viterbi_pruned -c 1 -o gpurun_out/r2z_prof_vit python tools/profile_cases.py viterbi > /dev/null 2>&1
ncu -i gpurun_out/r2z_prof_vit.ncu-rep --page raw --csv > gpurun_out/r2z_vit_raw.csv 2>/dev/null
