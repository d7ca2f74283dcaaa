mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? >> gpurun_out/status.txt
B="python bench.py --steps 995 --warmup 5 --ncu 0 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10"
BH_FUSE_KEYS=1 timeout 600 $B > gpurun_out/keys_fused.log 2>&1
BH_FUSE_KEYS=0 timeout 600 $B > gpurun_out/keys_sep.log 2>&1
BH_FUSE_KEYS=1 timeout 600 $B > gpurun_out/keys_fused2.log 2>&1
BH_FUSE_KEYS=0 timeout 600 $B > gpurun_out/keys_sep2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_hilbert.py tests/test_gpu_f64.py -x -q -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
