mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="python bench.py --ncu 0 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10"
BH_INITIAL_RELABEL=0 timeout 900 $B --steps 20 --warmup 5 > gpurun_out/i0_early.log 2>&1
BH_INITIAL_RELABEL=1 timeout 900 $B --steps 20 --warmup 5 > gpurun_out/i1_early.log 2>&1
BH_INITIAL_RELABEL=0 timeout 900 $B > gpurun_out/i0_full.log 2>&1
BH_INITIAL_RELABEL=1 timeout 900 $B > gpurun_out/i1_full.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1
