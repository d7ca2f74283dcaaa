# chain knobs A/B: prebuilt variants build/<v>.so (tools/build_variant.py):
# microbench (sort / tree build + prefix summarize alone) and the
# full-schedule bench for each
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/ck_*
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? >> gpurun_out/status.txt
B="python bench.py --steps 995 --warmup 5 --ncu 0 --cpu-steps 0 --e2e-repeats 1 --stage-iters 10"
for v in base ${VARIANTS}; do
  L=""; [ "$v" != base ] && L="$PWD/build/$v.so"
  BH_LIB=$L timeout 600 python tools/microbench.py --preroll 600 --reps 20 > gpurun_out/ck_micro_$v.log 2>&1
  BH_LIB=$L timeout 600 $B > gpurun_out/ck_bench_$v.log 2>&1
done
echo done >> gpurun_out/status.txt
