# GPU call: bench (C3, default schedule, ncu child) + an ncu --set full capture
# of the fused force launch (and the separate traversal / sweep launches) at
# iteration ${IT:-600}; summaries land in gpurun_out/.
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? >> gpurun_out/status.txt
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status.txt
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"${NCU_K:-k_forces|k_repulsive|k_attractive}" -o gpurun_out/prof \
  python bench.py --ncu-child --config c3 --ncu-iteration ${IT:-600} > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$? >> gpurun_out/status.txt
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --ncu-child --config c3 --ncu-iteration ${IT:-600} > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$? >> gpurun_out/status.txt
