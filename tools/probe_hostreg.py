import time, numpy as np, torch, ctypes
cudart = ctypes.CDLL("libcudart.so.12") if False else None
x = np.ones((1_000_000, 128), np.float32)
d = torch.empty((1_000_000, 128), dtype=torch.float32, device="cuda")
cr = torch.cuda.cudart()
for rep in range(3):
    t = time.perf_counter()
    r = cr.cudaHostRegister(x.ctypes.data, x.nbytes, 0)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    src = torch.from_numpy(x)
    d.copy_(src, non_blocking=True); torch.cuda.synchronize()
    t2 = time.perf_counter()
    cr.cudaHostUnregister(x.ctypes.data)
    t3 = time.perf_counter()
    print(f"register {1e3*(t1-t):.1f} ms  copy {1e3*(t2-t1):.1f} ms  unregister {1e3*(t3-t2):.1f} ms  rc {r}")
