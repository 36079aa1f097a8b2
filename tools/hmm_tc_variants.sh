#!/bin/bash
# A/B the tensor-core HMM forward operand types / configurations at the full
# BASELINE config (4096 signals x 10^4 steps x 1024 states), plus precision.
for v in f16 tf32 f16s6 f16c1; do
  PMX_HMM_TC=$v timeout 300 python bench.py --steps 2 --warmup 3 --case hmm_forward --no-cpu \
    > gpurun_out/bench_hmm_$v.json 2>gpurun_out/bench_hmm_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_hmm_$v.json').read().strip().splitlines()[-1]); k=d['case_studies']['hmm_forward']; print('$v', k.get('ms_per_step'), k.get('error'))"
  PMX_HMM_TC=$v timeout 300 python tools/hmm_precision.py 1024 2000 64
done
