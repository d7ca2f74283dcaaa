# ncu --set full of one iteration's tree chain (microbench state at iteration 600)
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? >> gpurun_out/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_morton|k_sort|k_tree|k_prefix|k_summarize_prefix" --launch-skip 20 -c 10 -o gpurun_out/prof_chain python tools/microbench.py --preroll 600 --reps 1 > gpurun_out/ncu_chain.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
