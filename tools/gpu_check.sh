# GPU suite (C3 parity excluded unless its fixture exists) + a C3 bench line
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? >> gpurun_out/status.txt
SEL=""; [ -f tests/golden/c3_run.npz ] || SEL="--deselect tests/test_gpu_c3.py"
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider $SEL > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 900 python bench.py ${BENCH_ARGS:---cpu-steps 0 --e2e-repeats 1} > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status.txt
