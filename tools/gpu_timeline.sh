# GPU timeline of the fast path at C3 (torch.profiler / CUPTI)
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? >> gpurun_out/status.txt
timeout 900 python tools/timeline.py --preroll ${PRE:-600} --iters 10 --out gpurun_out/timeline.json > gpurun_out/timeline.log 2>&1; echo timeline=$? >> gpurun_out/status.txt
