mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python tools/build_variant.py build/old64.so --src=forces_f64.cu=tools/_f64_old.cu > gpurun_out/bvar.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "f64 or multirank" > gpurun_out/pytest_f64.log 2>&1; echo rc=$? >> gpurun_out/pytest_f64.log
timeout 600 python tools/microbench.py --preroll 600 --reps 10 --precision f64 > gpurun_out/mb64_new.log 2>&1
BH_LIB=$PWD/build/old64.so timeout 600 python tools/microbench.py --preroll 600 --reps 10 --precision f64 > gpurun_out/mb64_old.log 2>&1
B="python bench.py --precision f64 --ncu 0 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10"
timeout 900 $B > gpurun_out/f64_new.log 2>&1
BH_LIB=$PWD/build/old64.so timeout 900 $B > gpurun_out/f64_old.log 2>&1
