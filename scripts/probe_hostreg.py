"""Probe: cost of cudaHostRegister / Unregister on a pageable numpy buffer (host drop-in design)."""
import time
import numpy as np
import torch
cr = torch.cuda.cudart()
torch.cuda.init()
for mb in (64, 256, 800):
    a = np.ones(mb << 17, dtype=np.int64)  # mb MB
    a[::512] = 2  # touch
    for rep in range(3):
        t0 = time.perf_counter()
        r = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
        t1 = time.perf_counter()
        r2 = cr.cudaHostUnregister(a.ctypes.data)
        t2 = time.perf_counter()
        print(f"{mb} MB: register {1e3 * (t1 - t0):.2f} ms ({a.nbytes / (t1 - t0) / 1e9:.1f} GB/s) "
              f"unregister {1e3 * (t2 - t1):.2f} ms rc={r},{r2}", flush=True)
x = np.ones(2_000_000_00 // 8 * 8, dtype=np.int64)
t0 = time.perf_counter(); y = x.copy(); t1 = time.perf_counter()
print(f"single-thread copy {x.nbytes / (t1 - t0) / 1e9:.1f} GB/s")
