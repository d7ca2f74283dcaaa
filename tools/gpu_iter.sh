# iteration loop: build, targeted GPU tests (PYK), microbench, timeline, bench
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? >> gpurun_out/status.txt
if [ -n "${PYK}" ]; then timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "${PYK}" > gpurun_out/pytest_k.log 2>&1; echo pytest_k=$? >> gpurun_out/status.txt; fi
timeout 900 python tools/microbench.py --preroll 600 --reps 20 > gpurun_out/micro.log 2>&1; echo micro=$? >> gpurun_out/status.txt
timeout 600 python tools/timeline.py --preroll 600 --iters 10 > gpurun_out/timeline.log 2>&1; echo tl=$? >> gpurun_out/status.txt
timeout 600 python bench.py --steps 995 --warmup 5 --ncu 0 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10 > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status.txt
if [ "${FULL:-0}" = "1" ]; then timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt; fi
if [ -n "${EXTRA}" ]; then timeout 1200 bash -c "${EXTRA}" > gpurun_out/extra.log 2>&1; echo extra=$? >> gpurun_out/status.txt; fi
