#!/bin/bash
# A/B the tensor-core HMM forward configurations at the full BASELINE config.
for v in 0 1 2 3; do
  PMX_HMM_TC_VARIANT=$v timeout 200 python bench.py --steps 2 --warmup 3 --case hmm_forward --cpu-seconds 1 \
    --no-cpu > gpurun_out/bench_hmm_v$v.json 2>gpurun_out/bench_hmm_v$v.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_hmm_v$v.json')); k=d['case_studies']['hmm_forward']; print('variant $v', k.get('ms_per_step'), k.get('error'))"
done
