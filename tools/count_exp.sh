#!/bin/bash
# count-kernel timing experiments (TACO_COUNT_DBG skips phases; results are wrong by design)
for dbg in 0 2 3 4 6 7; do
  TACO_COUNT_DBG=$dbg python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cexp_$dbg.json 2>/dev/null
  python - "$dbg" <<'PY'
import json, sys
b = json.loads(open(f"gpurun_out/cexp_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("dbg", sys.argv[1], "k_count ms", b["path_roofline"]["kernels_ms"]["k_count"], "step", round(b["ms_per_step"], 3))
PY
done
