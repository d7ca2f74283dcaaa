# A/B of the CSR sweep layout (strided lanes vs 4 contiguous entries per
# lane) and the per-row column sort at relabel
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? >> gpurun_out/status.txt
python tools/build_variant.py build/contig.so -DBH_ATTR_STRIDED=0 > gpurun_out/bc.log 2>&1
B="python bench.py --steps 995 --warmup 5 --ncu 0 --cpu-steps 0 --e2e-repeats 1"
timeout 900 $B > gpurun_out/ab_strided_sorted.log 2>&1
BH_SORT_ROWS=0 timeout 900 $B > gpurun_out/ab_strided_unsorted.log 2>&1
BH_LIB=$PWD/build/contig.so timeout 900 $B > gpurun_out/ab_contig_sorted.log 2>&1
BH_LIB=$PWD/build/contig.so BH_SORT_ROWS=0 timeout 900 $B > gpurun_out/ab_contig_unsorted.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
