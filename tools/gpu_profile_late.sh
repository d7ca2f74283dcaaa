# tests + late-iteration ncu captures of the two force kernels
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 900 python tools/microbench.py --preroll 600 --reps 5 > gpurun_out/micro.log 2>&1; echo micro=$? >> gpurun_out/status.txt
timeout 900 ncu --target-processes all --set full --clock-control none --import-source on -k regex:k_attractive -c 1 -o gpurun_out/prof_att python tools/microbench.py --preroll 600 --reps 1 > gpurun_out/ncu_att.log 2>&1; echo ncu_att=$? >> gpurun_out/status.txt
timeout 900 ncu --target-processes all --set full --clock-control none --import-source on -k regex:k_repulsive -c 1 -o gpurun_out/prof_rep python tools/microbench.py --preroll 600 --reps 1 > gpurun_out/ncu_rep.log 2>&1; echo ncu_rep=$? >> gpurun_out/status.txt
