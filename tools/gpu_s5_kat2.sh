mkdir -p gpurun_out; rm -f gpurun_out/status.txt
timeout 900 python -m pytest tests/test_gpu_kat2.py -m gpu -q -p no:cacheprovider > gpurun_out/kat2.log 2>&1; echo kat2=$? >> gpurun_out/status.txt
