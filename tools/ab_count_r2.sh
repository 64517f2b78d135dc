bash tools/ab_variants.sh 10 skiphalf nopair
for e in "TACO_CLUSTER_IDS=196608" "TACO_CLUSTER_IDS=196608 TACO_COUNT_NT=512" "TACO_COUNT_NT=512" "TACO_CLUSTER_IDS=98304"; do
  env $e timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ab_env.json 2>gpurun_out/ab_env.err
  python - "$e" <<'PY'
import json, sys
try:
    b = json.loads(open("gpurun_out/ab_env.json").read().strip().splitlines()[-1])
    k = b["path_roofline"]["kernels_ms"]
    print(f"{sys.argv[1]:40s} qps {b['value']:9.0f} count {k['k_count']:.3f} rerank {k['k_rerank']:.3f} recall {b['config']['recall@10']}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
TACO_LIB_VARIANT=build/variants/skiphalf.so python -m pytest tests -m gpu -x -q 2>&1 | tail -2
