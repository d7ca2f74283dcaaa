# knob sweep on the full C3 schedule (bench, no ncu/cpu/e2e extras)
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="python bench.py --steps 995 --warmup 5 --ncu 0 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10"
for r in ${RELABELS:-25 50 100}; do timeout 600 $B --relabel-every $r > gpurun_out/knob_relabel_$r.log 2>&1; done
