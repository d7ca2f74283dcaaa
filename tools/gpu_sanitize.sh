mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python tools/attr_dedup.py --preroll 600 > gpurun_out/dedup.log 2>&1; echo dedup=$? >> gpurun_out/status.txt
for tool in memcheck racecheck synccheck initcheck; do
  BH_SAN_N=768 BH_SAN_ITERS=14 timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/san_$tool.log 2>&1; echo san_$tool=$? >> gpurun_out/status.txt
done
timeout 900 python -m pytest tests/test_gpu_c4.py -q -s -p no:cacheprovider > gpurun_out/pytest_c4.log 2>&1; echo c4=$? >> gpurun_out/status.txt
