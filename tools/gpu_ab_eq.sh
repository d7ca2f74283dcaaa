# A/B with bitwise trajectory check: base build vs VARIANT (-D flags)
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? >> gpurun_out/status.txt
python tools/build_variant.py build/var.so ${VARIANT} > gpurun_out/bvar.log 2>&1
python tools/traj_dump.py gpurun_out/ya.npy > gpurun_out/traja.log 2>&1
BH_LIB=$PWD/build/var.so python tools/traj_dump.py gpurun_out/yb.npy > gpurun_out/trajb.log 2>&1
python -c "
import numpy as np
for t in ('0.5','0.8'):
    a=np.load(f'gpurun_out/ya_t{t}.npy'); b=np.load(f'gpurun_out/yb_t{t}.npy')
    print(t, 'base==variant', np.array_equal(a,b))
" > gpurun_out/equiv.txt 2>&1
rm -f gpurun_out/*.npy
B="python bench.py --steps 995 --warmup 5 --ncu 0 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10"
timeout 600 python tools/microbench.py --preroll 600 --reps 20 > gpurun_out/ab_base_micro.log 2>&1
timeout 600 $B > gpurun_out/ab_base_bench.log 2>&1
BH_LIB=$PWD/build/var.so timeout 600 python tools/microbench.py --preroll 600 --reps 20 > gpurun_out/ab_var_micro.log 2>&1
BH_LIB=$PWD/build/var.so timeout 600 $B > gpurun_out/ab_var_bench.log 2>&1
if [ -n "${PYK}" ]; then timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "${PYK}" > gpurun_out/pytest_k.log 2>&1; echo pytest_k=$? >> gpurun_out/status.txt; fi
