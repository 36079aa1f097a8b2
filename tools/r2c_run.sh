# r2c: TMEM read-bandwidth probe (+ the F16-accumulator TMEM layout check, separate process)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2211_00621_b200/csrc -lcuda -o /tmp/tmem_probe tools/tmem_probe.cu \
  && timeout 120 /tmp/tmem_probe > gpurun_out/tmem_probe.json 2> gpurun_out/tmem_probe.err
timeout 60 /tmp/tmem_probe layout > gpurun_out/tmem_layout.json 2>&1
cat gpurun_out/tmem_probe.json
