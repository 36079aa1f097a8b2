# r2x: ncu source pages of k_viterbi_pruned, k_hmm_fwd_quad and k_nn_grad (hot-instruction scan)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_viterbi_pruned -c 1 -o gpurun_out/r2x_prof_vit python tools/profile_cases.py viterbi > /dev/null 2>&1
ncu -i gpurun_out/r2x_prof_vit.ncu-rep --page source --csv > gpurun_out/r2x_vit_source.csv 2>/dev/null
ncu -i gpurun_out/r2x_prof_vit.ncu-rep --page raw --csv > gpurun_out/r2x_vit_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nn_grad -c 1 -o gpurun_out/r2x_prof_nn python tools/profile_cases.py nn > /dev/null 2>&1
ncu -i gpurun_out/r2x_prof_nn.ncu-rep --page source --csv > gpurun_out/r2x_nn_source.csv 2>/dev/null
ncu -i gpurun_out/r2x_prof_nn.ncu-rep --page raw --csv > gpurun_out/r2x_nn_raw.csv 2>/dev/null
ls gpurun_out | grep r2x
