# the GPU suite against the BH_DEBUG build (device-side invariant traps)
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? >> gpurun_out/status.txt
python tools/build_variant.py build/libbhtsne_b200_debug.so -DBH_DEBUG > gpurun_out/build_dbg.log 2>&1; echo build_dbg=$? >> gpurun_out/status.txt
BH_LIB=$PWD/build/libbhtsne_b200_debug.so timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_c3.py > gpurun_out/pytest_debug.log 2>&1; echo pytest_debug=$? >> gpurun_out/status.txt
BH_LIB=$PWD/build/libbhtsne_b200_debug.so timeout 900 python bench.py --steps 200 --warmup 5 --ncu 0 --cpu-steps 0 --e2e-repeats 1 > gpurun_out/bench_debug.log 2>&1; echo bench_debug=$? >> gpurun_out/status.txt
