set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in 1 2 3 4; do
  timeout 900 python bench.py --config $c > gpurun_out/s4_bench_cfg$c.json 2> gpurun_out/s4_bench_cfg$c.err
  python - $c <<'PY'
import json, sys
c = sys.argv[1]
try:
    b = json.loads(open(f"gpurun_out/s4_bench_cfg{c}.json").read().strip().splitlines()[-1])
    k = b["path_roofline"]["kernels_ms"]
    print(f"cfg{c} qps {b['value']:9.0f} e2e {b['e2e']['value']:9.0f} count {k['k_count']:.3f} rerank {k['k_rerank']:.3f} trav {k['k_traverse']:.3f} build {b['build_seconds']:.3f} recall {b['config']['recall@10']} frac {b['roofline']['frac']:.3f} cpu {b.get('cpu_baseline')}")
except Exception as e:
    print(c, "FAILED", e)
PY
done
TACO_GLOBAL_CHUNK=131072 timeout 900 python bench.py --config 4 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
b=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=b['path_roofline']['kernels_ms']; print('cfg4 chunk128K', round(b['value']), k['k_count'], k['k_rerank'])"
