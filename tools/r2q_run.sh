# r2q: ncu --set full of the k-mer pair kernel (T = 100)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kmer_fwd_pair -s 1 -c 1 -o gpurun_out/r2q_prof_kmer python tools/profile_cases.py kmer > gpurun_out/r2q_ncu.log 2>&1
ncu -i gpurun_out/r2q_prof_kmer.ncu-rep --page raw --csv > gpurun_out/r2q_kmer_raw.csv 2>/dev/null
ncu -i gpurun_out/r2q_prof_kmer.ncu-rep --page source --csv > gpurun_out/r2q_kmer_source.csv 2>/dev/null
tail -3 gpurun_out/r2q_ncu.log
