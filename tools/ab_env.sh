#!/bin/bash
# A/B environment settings on the config-2 bench (GPU box):  tools/ab_env.sh "A=1" "B=2 C=3" ...
mkdir -p gpurun_out
for e in "$@"; do
  env $e timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ab_env.json 2>gpurun_out/ab_env.err
  python - "$e" <<'PY'
import json, sys
try:
    b = json.loads(open("gpurun_out/ab_env.json").read().strip().splitlines()[-1])
    k = b["path_roofline"]["kernels_ms"]
    print(f"{sys.argv[1]:40s} qps {b['value']:9.0f} e2e {b['e2e']['value']:9.0f} count {k['k_count']:.3f} rerank {k['k_rerank']:.3f} trav {k['k_traverse']:.3f} recall {b['config']['recall@10']}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
