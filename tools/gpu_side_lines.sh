# final-tree side lines: the multi-GPU bench path on one GPU, the C4 kernel microbench, C3 in f64
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
BH_BENCH_SHARD1=1 timeout 900 python bench.py --steps 20 --warmup 5 --cpu-steps 0 --e2e-repeats 1 --ncu 0 > gpurun_out/bench_shard1.log 2>&1; echo shard1=$? >> gpurun_out/status.txt
timeout 1500 python bench.py --config c4 --cpu-steps 0 > gpurun_out/bench_c4.log 2>&1; echo c4=$? >> gpurun_out/status.txt
timeout 1200 python bench.py --precision f64 --cpu-steps 0 --e2e-repeats 1 --ncu 0 > gpurun_out/bench_f64.log 2>&1; echo f64=$? >> gpurun_out/status.txt
