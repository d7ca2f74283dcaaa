# A/B of the sub-warp traversal: SUB=16 (build) vs SUB=32 / 8 variants --
# bitwise trajectories and traversal timings
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? >> gpurun_out/status.txt
python tools/build_variant.py build/sub32.so -DBH_REP_SUB=32 > gpurun_out/b32.log 2>&1
python tools/build_variant.py build/sub8.so -DBH_REP_SUB=8 > gpurun_out/b8.log 2>&1
python tools/traj_dump.py gpurun_out/y16.npy > gpurun_out/traj16.log 2>&1
BH_LIB=$PWD/build/sub32.so python tools/traj_dump.py gpurun_out/y32.npy > gpurun_out/traj32.log 2>&1
BH_LIB=$PWD/build/sub8.so python tools/traj_dump.py gpurun_out/y8.npy > gpurun_out/traj8.log 2>&1
python -c "
import numpy as np
for t in ('0.5','0.8'):
    a=np.load(f'gpurun_out/y16_t{t}.npy'); b=np.load(f'gpurun_out/y32_t{t}.npy'); c=np.load(f'gpurun_out/y8_t{t}.npy')
    print(t, 'sub16==sub32', np.array_equal(a,b), 'sub8==sub32', np.array_equal(c,b))
" > gpurun_out/equiv.txt 2>&1
rm -f gpurun_out/*.npy
for v in 16 32 8; do
  if [ $v = 16 ]; then L=""; else L="BH_LIB=$PWD/build/sub$v.so"; fi
  env $L timeout 600 python tools/hilbert_probe.py > gpurun_out/probe_$v.log 2>&1
  env $L timeout 900 python bench.py --steps 995 --warmup 5 --ncu 0 --cpu-steps 0 --e2e-repeats 1 > gpurun_out/bench_$v.log 2>&1
done
