# r2u: seqLoop JIT kernel with 4 elements per thread per pass: parity tests + timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_skeletons.py -x -q -p no:cacheprovider > gpurun_out/pytest_seq.log 2>&1
tail -2 gpurun_out/pytest_seq.log
timeout 300 python tools/seq_ab.py > gpurun_out/seq_ab.log 2>&1; cat gpurun_out/seq_ab.log
