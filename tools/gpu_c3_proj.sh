mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_c3.py -v -s -p no:cacheprovider > gpurun_out/pytest_c3.log 2>&1; echo c3=$? > gpurun_out/status.txt
timeout 1200 python tools/multigpu_projection.py > gpurun_out/proj.log 2>&1; echo proj=$? >> gpurun_out/status.txt
