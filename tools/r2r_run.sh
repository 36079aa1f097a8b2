# r2r: k-mer pair kernel: parity, step time, and a clock64 trace of one cluster
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "kmer" > gpurun_out/pytest_kmer.log 2>&1
tail -1 gpurun_out/pytest_kmer.log
(timeout 300 python tools/kmer_time.py 1000; PMX_KMER_TRACE=1 timeout 300 python tools/kmer_time.py 300) > gpurun_out/kmer_time.log 2>&1
cat gpurun_out/kmer_time.log
