# r2s: k-mer pair kernel: step time, ncu
mkdir -p gpurun_out
timeout 300 python tools/kmer_time.py 1000 > gpurun_out/kmer_time.log 2>&1
cat gpurun_out/kmer_time.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kmer_fwd_pair -s 1 -c 1 -o gpurun_out/r2s_prof_kmer python tools/profile_cases.py kmer > gpurun_out/r2s_ncu.log 2>&1
ncu -i gpurun_out/r2s_prof_kmer.ncu-rep --page raw --csv > gpurun_out/r2s_kmer_raw.csv 2>/dev/null
ncu -i gpurun_out/r2s_prof_kmer.ncu-rep --page source --csv > gpurun_out/r2s_kmer_source.csv 2>/dev/null
