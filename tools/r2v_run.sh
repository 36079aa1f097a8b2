# r2v: ncu --set full of the k-NN tensor-core kernel at the full config (k_knn_tc only, not the prep kernels)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc -c 1 -o gpurun_out/r2v_prof_knn python tools/profile_cases.py knn_full > gpurun_out/r2v_ncu.log 2>&1
ncu -i gpurun_out/r2v_prof_knn.ncu-rep --page raw --csv > gpurun_out/r2v_knn_raw.csv 2>/dev/null
ncu -i gpurun_out/r2v_prof_knn.ncu-rep --page source --csv > gpurun_out/r2v_knn_source.csv 2>/dev/null
tail -2 gpurun_out/r2v_ncu.log
