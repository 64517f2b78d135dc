"""Per-kernel timeline of one index build (CUPTI via torch.profiler).

    python tools/prof_build.py [cfg]

Prints wall stages, per-kernel total/count, and the GPU busy union (the
build runs 2*N_s k-means halves on concurrent streams, so kernel sums
over-count; the union is the occupied GPU time)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_2603_24919_b200 as T  # noqa: E402
from paper_2603_24919_b200.workloads import make_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
X, Q, meta = make_config(cfg, nq=16)
P = T.IndexParams(meta["n_sub"], meta["s"], meta["clusters"], meta["kmeans_iters"], meta["seed"])
T.build_index(X, P)                       # warm (module load, allocations)
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    idx = T.build_index(X, P)
    wall = time.perf_counter() - t0
md = {k: v for k, v in idx.metadata.items() if k.endswith("seconds")}
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in evs)
agg = {}
for s, e, nm in iv:
    a = agg.setdefault(nm[:60], [0.0, 0])
    a[0] += (e - s) / 1e3
    a[1] += 1
busy, cur_s, cur_e = 0.0, None, None
for s, e, _ in iv:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
if cur_e is not None:
    busy += cur_e - cur_s
span = (iv[-1][1] - iv[0][0]) / 1e3 if iv else 0
print(json.dumps({"cfg": cfg, "wall_s": wall, "stages": md, "gpu_busy_ms": busy / 1e3,
                  "gpu_span_ms": span, "launches": len(iv)}, indent=1))
for nm, (ms, c) in sorted(agg.items(), key=lambda t: -t[1][0])[:30]:
    print(f"{ms:10.3f} ms {c:6d}  {nm}")
# per-stream windows (chrome trace carries the stream id)
import os, tempfile  # noqa: E402
tf = tempfile.mktemp(suffix=".json")
prof.export_chrome_trace(tf)
tr = json.load(open(tf))
os.unlink(tf)
per = {}
for ev in tr.get("traceEvents", []):
    if ev.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in ev:
        sid = ev.get("args", {}).get("stream", -1)
        a = per.setdefault(sid, [1e30, 0, 0.0, 0])
        a[0] = min(a[0], ev["ts"]); a[1] = max(a[1], ev["ts"] + ev["dur"]); a[2] += ev["dur"]; a[3] += 1
t0s = min(v[0] for v in per.values()) if per else 0
for sid, (a, b, busy_us, c) in sorted(per.items(), key=lambda t: t[1][0]):
    print(f"stream {sid}: [{(a - t0s) / 1e3:8.2f}, {(b - t0s) / 1e3:8.2f}] ms  busy {busy_us / 1e3:8.2f} ms  {c} ops")
# busy union per 10 ms window, to see idle gaps
if iv:
    t00 = iv[0][0]
    win = {}
    for s, e, _ in iv:
        b = int((s - t00) / 10000)
        win[b] = win.get(b, 0) + (e - s) / 1e3
    print("kernel-ms per 10 ms window:", [round(win.get(b, 0), 1) for b in range(max(win) + 1)])
# cluster-size skew (the Lloyd sums are one dependent add chain per cluster)
try:
    for j, sub in enumerate(idx.subspaces[:2]):
        for nm in ("codebook1", "codebook2"):
            a = getattr(sub, nm).assignments
            if a is not None:
                bc = np.bincount(np.asarray(a), minlength=meta["kprime"])
                print(f"sub {j} {nm}: cluster sizes max {bc.max()} mean {bc.mean():.0f} min {bc.min()}")
except Exception as ex:  # noqa: BLE001
    print("cluster sizes unavailable:", ex)
