#!/bin/bash
# r2 evidence run on one B200 (gpurun): L2 probe, ncu captures of RK4 (FP64 pipe
# counts for the roofline), the pruned Viterbi kernel, the k-mer kernel (DRAM
# traffic) and the HMM quad kernel; all under gpurun_out/.
set -x
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/l2_probe tools/l2_probe.cu && \
  /tmp/l2_probe > gpurun_out/l2_probe.json 2> gpurun_out/l2_probe.log
for c in rk4 viterbi kmer hmm; do
  case $c in
    rk4) k=k_rk4 ;; viterbi) k=k_viterbi_pruned ;; kmer) k=k_kmer_fwd ;; hmm) k=k_hmm_fwd_quad ;;
  esac
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
    -o gpurun_out/r2_prof_$c python tools/profile_cases.py $c > gpurun_out/r2_prof_$c.log 2>&1
  ncu -i gpurun_out/r2_prof_$c.ncu-rep --page raw --csv > gpurun_out/r2_${c}_raw.csv 2>/dev/null
done
ls -la gpurun_out
