for f in gpurun_out/ck_bench_*.log; do n=${f#gpurun_out/ck_bench_}; n=${n%.log}; echo "== $n";
tail -1 gpurun_out/ck_micro_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v,4) for k,v in d.items() if k in ('sort_ms','sort_build_ms','tree_build_prefix_ms','summarize_prefix_ms','step_fused_ms','step_traversal_ms')})";
tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', round(d['value'],1), {k: round(v,4) for k,v in d['stage_ms'].items() if k in ('tree','summarize','iteration_pipelined','force_phase_pipelined')})"; done
