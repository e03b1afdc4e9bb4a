"""Cost of cudaHostRegister / Unregister for plan-sized host arrays vs a
staged copy (decides whether one-shot uploads should pin the caller's arrays)."""
import ctypes
import time

import numpy as np
import torch

rt = ctypes.CDLL("libcudart.so.12") if False else None
torch.cuda.init()
cudart = torch.cuda.cudart()
for mb in (8, 64, 125, 250):
    a = np.ones(mb * (1 << 20) // 8)
    d = torch.empty(a.size, dtype=torch.float64, device="cuda")
    for rep in range(3):
        t0 = time.perf_counter()
        r = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        d.copy_(torch.from_numpy(a), non_blocking=True)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        cudart.cudaHostUnregister(a.ctypes.data)
        t4 = time.perf_counter()
        tp = time.perf_counter()
        d.copy_(torch.from_numpy(a))
        torch.cuda.synchronize()
        t5 = time.perf_counter()
        print(f"{mb} MB: register {1e3*(t1-t0):.2f} ms (rc {r}), H2D pinned {1e3*(t3-t2):.2f} ms "
              f"({a.nbytes/(t3-t2)/1e9:.1f} GB/s), unregister {1e3*(t4-t3):.2f} ms, pageable H2D {1e3*(t5-tp):.2f} ms "
              f"({a.nbytes/(t5-tp)/1e9:.1f} GB/s)", flush=True)
