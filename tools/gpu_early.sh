# the driver's window (iterations 5-25): stage breakdown, ncu of iteration 15
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --ncu-iteration 15 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10 > gpurun_out/early.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --ncu 0 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10 --relabel-every 10 > gpurun_out/early_r10.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --ncu 0 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10 --relabel-every 5 > gpurun_out/early_r5.log 2>&1
timeout 900 python bench.py --steps 200 --warmup 300 --ncu 0 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10 > gpurun_out/late.log 2>&1
