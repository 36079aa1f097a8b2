# r2f: k-NN pair kernel: parity tests, probes, bench line, ncu
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "knn" > gpurun_out/pytest_knn.log 2>&1
tail -3 gpurun_out/pytest_knn.log
for p in 0; do PMX_KNN_PROBE=$p timeout 300 python tools/knn_time.py; done > gpurun_out/knn_probe.log 2>&1
cat gpurun_out/knn_probe.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --case knn > gpurun_out/bench_knn.json 2> gpurun_out/bench_knn.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_knn.json').read().strip().splitlines()[-1]); k=d['case_studies']['knn']; print('knn ms', k.get('ms_per_step'), k.get('roofline',{}).get('frac'), k.get('parity'))"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc -c 1 -o gpurun_out/r2f_prof_knn python tools/profile_cases.py knn_full > gpurun_out/r2f_prof_knn.log 2>&1
ncu -i gpurun_out/r2f_prof_knn.ncu-rep --page raw --csv > gpurun_out/r2f_knn_raw.csv 2>/dev/null
ncu -i gpurun_out/r2f_prof_knn.ncu-rep --page source --csv --print-source sass > gpurun_out/r2f_knn_source.csv 2>/dev/null
