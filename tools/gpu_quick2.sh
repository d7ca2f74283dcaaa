# quick GPU check: hilbert tests, multirank, bench (20 steps + full)
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? >> gpurun_out/status.txt
timeout 900 python -m pytest tests/test_gpu_hilbert.py tests/test_gpu_multirank.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 900 python bench.py --steps 20 --warmup 5 --ncu 0 --cpu-steps 0 > gpurun_out/bench_c3.log 2>&1; echo bench=$? >> gpurun_out/status.txt
timeout 900 python bench.py --ncu 0 --cpu-steps 0 > gpurun_out/bench_c3_full.log 2>&1; echo bench_full=$? >> gpurun_out/status.txt
