"""Cost of cudaHostRegister on a query batch vs a copy into pinned memory."""
import time

import numpy as np
import torch

Q = np.random.default_rng(0).random((10000, 128), dtype=np.float32)
pin = torch.empty((10000, 128), dtype=torch.float32, pin_memory=True)
dev = torch.empty((10000, 128), dtype=torch.float32, device="cuda")
rt = torch.cuda.cudart()
for _ in range(3):
    np.copyto(pin.numpy(), Q)
t0 = time.perf_counter()
for _ in range(20):
    np.copyto(pin.numpy(), Q)
    dev.copy_(pin, non_blocking=True)
    torch.cuda.synchronize()
print("copy into pinned + H2D: %.3f ms" % ((time.perf_counter() - t0) / 20 * 1e3))
t0 = time.perf_counter()
for _ in range(20):
    rt.cudaHostRegister(Q.ctypes.data, Q.nbytes, 0)
    dev.copy_(torch.from_numpy(Q), non_blocking=True)
    torch.cuda.synchronize()
    rt.cudaHostUnregister(Q.ctypes.data)
print("register + H2D + unregister: %.3f ms" % ((time.perf_counter() - t0) / 20 * 1e3))
t0 = time.perf_counter()
for _ in range(20):
    dev.copy_(torch.from_numpy(Q), non_blocking=True)
    torch.cuda.synchronize()
print("pageable H2D: %.3f ms" % ((time.perf_counter() - t0) / 20 * 1e3))
