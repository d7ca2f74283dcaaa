# Final-tree evidence: GPU suite, smoke, the default bench line (full schedule), the driver's window for both arms
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
(time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider) > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
(time timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5) > gpurun_out/bench_ref_drv.log 2>&1; echo ref=$? >> gpurun_out/status.txt
(time timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5) > gpurun_out/bench_drv.log 2>&1; echo benchdrv=$? >> gpurun_out/status.txt
(time timeout 1200 python bench.py) > gpurun_out/bench_c3.log 2>&1; echo bench=$? >> gpurun_out/status.txt
(time timeout 900 python tools/run_bench.py c3) > gpurun_out/run_c3.log 2>&1; echo run_c3=$? >> gpurun_out/status.txt
timeout 600 python tools/knn_bench.py c3 --f64 > gpurun_out/knn_c3_f64.log 2>&1; echo knn_f64=$? >> gpurun_out/status.txt
