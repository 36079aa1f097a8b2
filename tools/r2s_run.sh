# r2s: k-mer pair kernel: step time, trace build, ncu
mkdir -p gpurun_out
timeout 300 python tools/kmer_time.py 1000 > gpurun_out/kmer_time.log 2>&1
PMX_B200_LIB=paper_2211_00621_b200/libpmx_kmer_trace.so PMX_KMER_TRACE=1 timeout 300 python tools/kmer_time.py 300 >> gpurun_out/kmer_time.log 2>&1
grep -v "^cta" gpurun_out/kmer_time.log; grep "g=20[45]" gpurun_out/kmer_time.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kmer_fwd_pair -s 1 -c 1 -o gpurun_out/r2s_prof_kmer python tools/profile_cases.py kmer > gpurun_out/r2s_ncu.log 2>&1
ncu -i gpurun_out/r2s_prof_kmer.ncu-rep --page raw --csv > gpurun_out/r2s_kmer_raw.csv 2>/dev/null
ncu -i gpurun_out/r2s_prof_kmer.ncu-rep --page source --csv > gpurun_out/r2s_kmer_source.csv 2>/dev/null
