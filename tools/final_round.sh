#!/bin/bash
# Round-end measurement pass on the GPU box: tests, smoke, the four config bench lines,
# the experiment-knob sanity lines and the ncu captures (tools/final_ncu.sh).
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
bash tools/run_cfgs.sh > gpurun_out/final_cfgs.log 2>&1
grep "^cfg\|passed\|failed" gpurun_out/final_cfgs.log | cut -c1-140
tools/ab_env.sh TACO_COUNT_PG=0 TACO_COUNT_NT=512 TACO_COUNT_NT=1024 TACO_FUSED=1 TACO_TRAVERSE=smem
tools/final_ncu.sh > gpurun_out/final_ncu.log 2>&1
ls gpurun_out/*.ncu-rep
