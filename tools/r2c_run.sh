# r2c: TMEM layout checks (F16 accumulator, .pack::16b loads)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2211_00621_b200/csrc -lcuda -o /tmp/tmem_probe tools/tmem_probe.cu \
  && timeout 60 /tmp/tmem_probe layout > gpurun_out/tmem_layout.json 2>&1
cat gpurun_out/tmem_layout.json | cut -c1-1200
