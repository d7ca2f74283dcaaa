# relabel interval A/B on the full schedule
mkdir -p gpurun_out; rm -f gpurun_out/rl_*
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="python bench.py --steps 995 --warmup 5 --ncu 0 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10"
for r in ${INTERVALS:-50 100 200 50}; do
  timeout 600 $B --relabel-every $r > gpurun_out/rl_$r.log 2>&1
  tail -1 gpurun_out/rl_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($r, round(d['value'],1), round(d['e2e']['value'],1))" >> gpurun_out/rl_summary.txt
done
