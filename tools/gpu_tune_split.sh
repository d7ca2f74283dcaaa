# side-sweep share A/B: full schedule and the driver's window
mkdir -p gpurun_out
B="python bench.py --ncu 0 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10"
for s in 0.25 0.275 0.3; do timeout 600 $B --steps 995 --warmup 5 --attr-split $s > gpurun_out/tune_split_$s.log 2>&1; done
for s in 0.275 0.3 0.325 0.35; do for rep in a b; do timeout 600 $B --steps 20 --warmup 5 --attr-split $s > gpurun_out/tune_drv_${s}_$rep.log 2>&1; done; done
