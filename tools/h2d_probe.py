"""Host->device transfer options on this box: pinned DMA, pageable DMA, cudaHostRegister."""
import ctypes
import time

import numpy as np
import torch

cudart = ctypes.CDLL("libcudart.so.12") if False else None
n = 150_000_000  # 1.2 GB of float64
a = np.random.default_rng(0).random(n)
d = torch.empty(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()


def timed(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best


t_page = timed(lambda: d.copy_(torch.from_numpy(a), non_blocking=False))
pin = torch.empty(n, dtype=torch.float64).pin_memory()
pin.numpy()[:] = a
t_pin = timed(lambda: d.copy_(pin, non_blocking=True))
t_cpy = timed(lambda: np.copyto(pin.numpy(), a))
lib = ctypes.CDLL(torch.utils.cpp_extension.__file__.replace("cpp_extension.py", "") + "../lib/libcudart.so", mode=ctypes.RTLD_GLOBAL) if False else None
try:
    import cuda.bindings.runtime as rt
except Exception:
    from cuda import cudart as rt
t0 = time.perf_counter()
err = rt.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
t_reg = time.perf_counter() - t0
t_regcopy = timed(lambda: d.copy_(torch.from_numpy(a), non_blocking=True))
t0 = time.perf_counter()
rt.cudaHostUnregister(a.ctypes.data)
t_unreg = time.perf_counter() - t0
gb = a.nbytes / 1e9
print(f"1.2 GB: pageable H2D {gb / t_page:.1f} GB/s, pinned H2D {gb / t_pin:.1f} GB/s, host copy into pinned "
      f"{gb / t_cpy:.1f} GB/s (1 thread), register {1e3 * t_reg:.1f} ms ({err}), registered H2D {gb / t_regcopy:.1f} GB/s, "
      f"unregister {1e3 * t_unreg:.1f} ms")
