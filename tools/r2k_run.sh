# r2k: evidence refresh: full GPU tests, smoke, bench + reference arm, launch list, ncu of k_rk4 (angle-addition mode)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/r2k_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-parity > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rk4 -c 1 -o gpurun_out/r2k_prof_rk4 python tools/profile_cases.py rk4 > /dev/null 2>&1
ncu -i gpurun_out/r2k_prof_rk4.ncu-rep --page raw --csv > gpurun_out/r2k_rk4_raw.csv 2>/dev/null
ls gpurun_out | head -50
