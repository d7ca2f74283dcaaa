# quick GPU check: bench + launch list (no tests)
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
timeout 900 python bench.py --steps 995 --warmup 5 --cpu-steps 0 --e2e-steps 5 > gpurun_out/bench_c3.log 2>&1; echo bench=$? >> gpurun_out/status.txt
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-steps 0 --e2e-steps 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --kernel-name-base mangled -k regex:_ZN2bh --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --cpu-steps 0 --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$? >> gpurun_out/status.txt
