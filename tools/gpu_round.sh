# GPU call: tests, smoke, bench, reference arm, launch list, late-iteration ncu of the fused force kernel.
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo bench=$? >> gpurun_out/status.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$? >> gpurun_out/status.txt
if [ "${NCU:-1}" = "1" ]; then
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-steps 0 --e2e-steps 1 --e2e-repeats 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --kernel-name-base mangled -k regex:_ZN2bh --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --cpu-steps 0 --e2e-steps 1 --e2e-repeats 1 > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$? >> gpurun_out/status.txt
timeout 900 python tools/microbench.py --preroll 600 --reps 1 > gpurun_out/micro_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_forces}" -c 1 -o gpurun_out/prof python tools/microbench.py --preroll 600 --reps 1 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$? >> gpurun_out/status.txt
fi
