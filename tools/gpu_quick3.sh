mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? >> gpurun_out/status.txt
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_gpu_c3.py > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 900 python bench.py --ncu 1 --cpu-steps 0 > gpurun_out/bench_c3_full.log 2>&1; echo bench_full=$? >> gpurun_out/status.txt
