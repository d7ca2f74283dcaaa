mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="python bench.py --steps 995 --warmup 5 --ncu 0 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10"
timeout 600 $B > gpurun_out/k_default.log 2>&1
timeout 600 $B --no-fuse --attr-split 0.999 > gpurun_out/k_nofuse_side1.log 2>&1
timeout 600 $B --no-fuse --attr-split 0.6 > gpurun_out/k_nofuse_side06.log 2>&1
timeout 600 $B --no-fuse > gpurun_out/k_nofuse.log 2>&1
