# round-2 GPU call: build, full GPU suite, smoke, driver-shaped bench (both arms),
# default-schedule bench, launch list + ncu --set full of the force launches.
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? >> gpurun_out/status.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo ref=$? >> gpurun_out/status.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.log 2>&1; echo bench=$? >> gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench_c3_full.log 2>&1; echo bench_full=$? >> gpurun_out/status.txt
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"${NCU_K:-k_forces|k_repulsive|k_attractive}" -o gpurun_out/prof \
  python bench.py --ncu-child --config c3 --ncu-iteration ${IT:-600} > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$? >> gpurun_out/status.txt
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --ncu-child --config c3 --ncu-iteration ${IT:-600} > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$? >> gpurun_out/status.txt
