# r2m: Viterbi pruned kernel with one round of prefetch: parity tests + bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "viterbi" > gpurun_out/pytest_vit.log 2>&1
tail -3 gpurun_out/pytest_vit.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --case viterbi > gpurun_out/bench_vit.json 2> gpurun_out/bench_vit.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_vit.json').read().strip().splitlines()[-1]); k=d['case_studies']['viterbi']; print('viterbi ms', k.get('ms_per_step'), k.get('roofline',{}).get('frac'), k.get('parity'))"
