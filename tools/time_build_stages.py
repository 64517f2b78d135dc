"""Warm config-2 builds the way bench.py times them, with the covariance
stage split (DeviceIndex create / set_data / fit_covariance) from the
library's own timers (TACO_DEBUG_BUILD=1)."""
import os, sys, time, gc
sys.path.insert(0, "/root/repo")
import paper_2603_24919_b200 as T
from paper_2603_24919_b200 import engine
from paper_2603_24919_b200.workloads import make_config

X, Q, m = make_config(2, nq=16)
P = T.IndexParams(m["n_sub"], m["s"], m["clusters"], m["kmeans_iters"], m["seed"])
orig_call = engine.nat.call
acc = {}
def timed_call(name, *a):
    t = time.perf_counter()
    r = orig_call(name, *a)
    acc[name] = acc.get(name, 0.0) + time.perf_counter() - t
    return r
engine.nat.call = timed_call
orig_dev = engine.nat.DeviceIndex
def timed_dev(*a, **k):
    t = time.perf_counter()
    r = orig_dev(*a, **k)
    acc["DeviceIndex()"] = acc.get("DeviceIndex()", 0.0) + time.perf_counter() - t
    return r
engine.nat.DeviceIndex = timed_dev
idx = T.build_index(X, P)
for rep in range(4):
    idx = None
    gc.collect()
    acc.clear()
    t = time.perf_counter()
    idx = T.build_index(X, P)
    w = time.perf_counter() - t
    print(f"build {w*1e3:.1f} ms  " + "  ".join(f"{k} {v*1e3:.1f}" for k, v in sorted(acc.items(), key=lambda kv: -kv[1])[:8]))
    print("   metadata", {k: round(v * 1e3, 1) for k, v in idx.metadata.items() if k.endswith("seconds")})
