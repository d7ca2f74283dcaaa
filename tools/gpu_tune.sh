# knob sweep at C3: side-sweep share and fused CTA ratio
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="python bench.py --steps 995 --warmup 5 --ncu 0 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10"
for s in 0.25 0.3 0.35 0.4 0.45; do timeout 600 $B --attr-split $s > gpurun_out/tune_split_$s.log 2>&1; done
for r in 1.5 2.5 3; do BH_FUSE_RATIO=$r timeout 600 $B > gpurun_out/tune_ratio_$r.log 2>&1; done
