import torch, time
for n in (100, 356, 700, 1127):
    g = torch.randn(n, n, dtype=torch.complex128, device='cuda')
    l = torch.tril(g) * torch.exp(-torch.arange(n, device='cuda') / 20.0)
    h = l.conj().T @ l
    for drv in (None, 'syevj') if False else (None,):
        torch.linalg.eigh(h); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5): w, v = torch.linalg.eigh(h)
        torch.cuda.synchronize()
        print(f"torch.linalg.eigh n={n}: {(time.perf_counter()-t)/5*1e3:.2f} ms")
