# r2z: k-NN CTA-pair kernel (cta_group::2): parity tests + timing vs the single-CTA kernel
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "knn" > gpurun_out/pytest_knn.log 2>&1
tail -3 gpurun_out/pytest_knn.log
timeout 120 python tools/knn_time.py > gpurun_out/knn_time.log 2>&1; PMX_KNN_SINGLE=1 timeout 120 python tools/knn_time.py >> gpurun_out/knn_time.log 2>&1
cat gpurun_out/knn_time.log
