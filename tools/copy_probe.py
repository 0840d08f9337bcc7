"""Host<->device copy paths for value-semantics tensors (84 MB): pageable,
pinned, and cudaHostRegister around a pageable buffer."""
import time

import numpy as np
import torch

n = 84 * 1024 * 1024 // 8
dev = torch.empty(n, dtype=torch.float64, device="cuda")
page = np.ones(n)
pin = torch.empty(n, dtype=torch.float64).pin_memory()
cr = torch.cuda.cudart()


def t(f, reps=5):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


src_page = torch.from_numpy(page)
print("H2D pageable  %.2f GB/s" % (n * 8 / t(lambda: dev.copy_(src_page)) / 1e9))
print("H2D pinned    %.2f GB/s" % (n * 8 / t(lambda: dev.copy_(pin, non_blocking=True)) / 1e9))
print("D2H pageable  %.2f GB/s" % (n * 8 / t(lambda: src_page.copy_(dev)) / 1e9))
print("D2H pinned    %.2f GB/s" % (n * 8 / t(lambda: pin.copy_(dev, non_blocking=True)) / 1e9))


def reg_h2d():
    p = page.ctypes.data
    cr.cudaHostRegister(p, n * 8, 0)
    dev.copy_(src_page, non_blocking=True)
    torch.cuda.synchronize()
    cr.cudaHostUnregister(p)


print("H2D register+copy+unregister %.2f GB/s" % (n * 8 / t(reg_h2d) / 1e9))
fresh = lambda: np.empty(n)  # noqa: E731
print("np.empty + zero fill (value-initialised vector) %.2f GB/s" % (n * 8 / t(lambda: np.zeros(n)) / 1e9))
