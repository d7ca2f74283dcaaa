mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="python bench.py --steps 995 --warmup 5 --ncu 0 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10"
timeout 600 $B > gpurun_out/gap_base.log 2>&1
timeout 600 $B --chunk-graph > gpurun_out/gap_chunkgraph.log 2>&1
timeout 600 $B --chunk 50 > gpurun_out/gap_chunk50.log 2>&1
timeout 600 $B --relabel-every 100 > gpurun_out/gap_relabel100.log 2>&1
timeout 600 $B --relabel-every 25 > gpurun_out/gap_relabel25.log 2>&1
timeout 600 $B --chunk 100 --chunk-graph --relabel-every 100 > gpurun_out/gap_c100.log 2>&1
