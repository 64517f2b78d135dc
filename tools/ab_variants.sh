#!/bin/bash
# A/B the default library against build/variants/*.so on the config-2 bench (GPU box)
#   tools/ab_variants.sh [steps] [variant ...]
STEPS=${1:-10}; shift
VARS=${@:-$(ls build/variants/*.so 2>/dev/null | xargs -n1 basename | sed 's/\.so$//')}
mkdir -p gpurun_out
for v in default $VARS; do
  if [ $v = default ]; then E=""; else E="TACO_LIB_VARIANT=build/variants/$v.so"; fi
  env $E timeout 300 python bench.py --no-cpu-baseline --steps $STEPS > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    b = json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
    k = b["path_roofline"]["kernels_ms"]
    print(f"{v:10s} qps {b['value']:9.0f} e2e {b['e2e']['value']:9.0f} count {k['k_count']:.3f} rerank {k['k_rerank']:.3f} trav {k['k_traverse']:.3f} build {b['build_seconds']:.3f} recall {b['config']['recall@10']}")
except Exception as e:
    print(v, "FAILED", e)
PY
done
