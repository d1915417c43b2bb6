import torch, time
n = 805306368 // 8
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device='cuda')
for name, f in [('h2d', lambda: d.copy_(h, non_blocking=True)), ('d2h', lambda: h.copy_(d, non_blocking=True))]:
    f(); torch.cuda.synchronize(); t=time.perf_counter()
    for _ in range(3): f()
    torch.cuda.synchronize(); print(name, 3*n*8/(time.perf_counter()-t)/1e9, 'GB/s')
