# A/B of compile-time variants: VARIANTS="name:-DX=1 name2:-DY=2"; microbench + bench each
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? >> gpurun_out/status.txt
if [ -n "${PYK}" ]; then timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "${PYK}" > gpurun_out/pytest_k.log 2>&1; echo pytest_k=$? >> gpurun_out/status.txt; fi
B="python bench.py --steps 995 --warmup 5 --ncu 0 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10"
timeout 600 python tools/microbench.py --preroll 600 --reps 20 > gpurun_out/ab_base_micro.log 2>&1
timeout 600 $B > gpurun_out/ab_base_bench.log 2>&1
for v in ${VARIANTS}; do
  name=${v%%:*}; defs=${v#*:}
  python tools/build_variant.py build/$name.so ${defs//,/ } > gpurun_out/ab_${name}_build.log 2>&1
  BH_LIB=$PWD/build/$name.so timeout 600 python tools/microbench.py --preroll 600 --reps 20 > gpurun_out/ab_${name}_micro.log 2>&1
  BH_LIB=$PWD/build/$name.so timeout 600 $B > gpurun_out/ab_${name}_bench.log 2>&1
done
