#!/bin/bash
# Round-2 final ncu captures (GPU box): one kernel per run, reports into gpurun_out/
set -x
Q='regex:^k_(transform|csort|traverse|traverse_sh|count|count_pg|count_enc|count_genc|plan_sums|plan_scan|tile_map|q_u8|rerank_i8|rerank_async|topk|finalize|hist_reduce|select|emit_rec)'
python tools/prof_query.py 2 10000 2 > gpurun_out/f_pq2.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -k "$Q" -c 400 --csv --log-file gpurun_out/r2f_query_launches.csv python tools/prof_query.py 2 10000 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_count_pg --launch-skip 1 -c 1 -o gpurun_out/f_count2 python tools/prof_query.py 2 10000 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rerank_i8 --launch-skip 1 -c 1 -o gpurun_out/f_rerank2 python tools/prof_query.py 2 10000 2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_count_pg --launch-skip 1 -c 1 -o gpurun_out/f_count3 python tools/prof_query.py 3 1000 2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_rerank_async --launch-skip 1 -c 1 -o gpurun_out/f_rerank3 python tools/prof_query.py 3 1000 2 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_count_genc --launch-skip 1 -c 1 -o gpurun_out/f_count4 python tools/prof_query.py 4 2000 2 > /dev/null 2>&1
ls -la gpurun_out/
