# r2i: HMM forward step time vs number of clusters (L2 contention vs per-SM latency) + step trace
mkdir -p gpurun_out
for n in 4096 2048 1024 512; do timeout 300 python tools/hmm_time.py 1000 $n; done > gpurun_out/hmm_scale.log 2>&1
PMX_HMM_QUAD_TRACE=1 timeout 300 python tools/hmm_time.py 100 4096 >> gpurun_out/hmm_scale.log 2>&1
cat gpurun_out/hmm_scale.log
