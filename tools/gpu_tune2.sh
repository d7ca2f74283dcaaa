# knob re-check after the traversal trims: fused CTA ratio and side-sweep share
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="python bench.py --steps 995 --warmup 5 --ncu 0 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10"
timeout 600 $B > gpurun_out/t_base.log 2>&1
for r in 1.75 2.25 2.5; do BH_FUSE_RATIO=$r timeout 600 $B > gpurun_out/t_ratio_$r.log 2>&1; done
for sp in 0.3 0.4; do timeout 600 $B --attr-split $sp > gpurun_out/t_split_$sp.log 2>&1; done
timeout 600 $B > gpurun_out/t_base2.log 2>&1
