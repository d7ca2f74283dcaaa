# exact-kNN A/B: the dot-product filter (default) vs the difference filter (BH_KNN_TILE=0); bit-exactness tests first
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "knn" > gpurun_out/pytest_knn.log 2>&1; echo pytest_knn=$? >> gpurun_out/status.txt
timeout 600 python tools/knn_bench.py ${KNN_CONFIGS:-c1 c2 c3} > gpurun_out/knn_tile.log 2>&1; echo tile=$? >> gpurun_out/status.txt
BH_KNN_TILE=0 timeout 600 python tools/knn_bench.py ${KNN_CONFIGS:-c1 c2 c3} > gpurun_out/knn_diff.log 2>&1; echo diff=$? >> gpurun_out/status.txt
