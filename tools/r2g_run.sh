# r2g: seqLoop entry A/B (copy + pmx_seq_loop vs pmx_seq_loop_from)
mkdir -p gpurun_out
for s in 20 1 40; do timeout 300 python tools/seq_ab.py $s; done > gpurun_out/seq_ab.log 2>&1
cat gpurun_out/seq_ab.log
