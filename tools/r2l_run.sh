# r2l: k-NN with parked slow-path groups: parity + timing
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "knn" > gpurun_out/pytest_knn.log 2>&1
tail -3 gpurun_out/pytest_knn.log
timeout 300 python tools/knn_time.py > gpurun_out/knn_time.log 2>&1; cat gpurun_out/knn_time.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --case knn > gpurun_out/bench_knn.json 2> gpurun_out/bench_knn.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_knn.json').read().strip().splitlines()[-1]); k=d['case_studies']['knn']; print('knn ms', k.get('ms_per_step'), k.get('roofline',{}).get('frac'), k.get('parity'))"
