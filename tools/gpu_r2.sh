# round-2 GPU call: tests, smoke, driver-shaped bench (ours + reference arm)
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? >> gpurun_out/status.txt
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q -p no:cacheprovider > gpurun_out/pytest_multirank.log 2>&1; echo multirank=$? >> gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo ref=$? >> gpurun_out/status.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.log 2>&1; echo bench=$? >> gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench_c3_full.log 2>&1; echo bench_full=$? >> gpurun_out/status.txt
