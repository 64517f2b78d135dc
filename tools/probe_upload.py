"""Repeated staged uploads of config-2 X into one device index: host-copy
time per upload (TACO_DEBUG_UPLOAD) with and without GPU work / sleeps in
between, to find what slows the host copy in back-to-back builds."""
import os, sys, time
os.environ["TACO_DEBUG_UPLOAD"] = "1"
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2603_24919_b200 import _native as nat
from paper_2603_24919_b200.workloads import make_config
import torch

X, Q, m = make_config(2, nq=16)
dev = nat.DeviceIndex(X.shape[0], X.shape[1], m["n_sub"], m["s"], m["clusters"], m["kmeans_iters"])
def up(tag):
    t = time.perf_counter()
    nat.call("taco_index_set_data", dev.h, nat.ptr(X))
    print(tag, f"wall {1e3*(time.perf_counter()-t):.1f} ms", file=sys.stderr, flush=True)
for i in range(3):
    up("back-to-back")
for i in range(3):
    time.sleep(0.1); up("after sleep 100ms")
a = torch.randn(8192, 8192, device="cuda")
for i in range(3):
    for _ in range(20): a = a @ a; a = a / a.norm()
    torch.cuda.synchronize(); up("after 20 GEMMs")
Y = np.empty_like(X)
for i in range(3):
    Y[:] = X; up("after host copy of X")
import gc
for i in range(3):
    dev = None; gc.collect()
    dev = nat.DeviceIndex(X.shape[0], X.shape[1], m["n_sub"], m["s"], m["clusters"], m["kmeans_iters"])
    up("fresh DeviceIndex")
import paper_2603_24919_b200 as T
P = T.IndexParams(m["n_sub"], m["s"], m["clusters"], m["kmeans_iters"], m["seed"])
idx = T.build_index(X, P)
for i in range(2):
    up("after a build (old dev)")
for i in range(3):
    t = time.perf_counter(); idx = T.build_index(X, P); print("build", 1e3*(time.perf_counter()-t), file=sys.stderr)
