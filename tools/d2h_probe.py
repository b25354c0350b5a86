import torch, time
for mb in (0.33, 1.77, 4):
    n = int(mb * 1e6 / 4)
    d = torch.randn(n, device="cuda")
    h = torch.empty(n, pin_memory=True)
    for _ in range(5): h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50): h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 50
    hp = torch.empty(n)
    t0 = time.perf_counter()
    for _ in range(50): hp.copy_(d); torch.cuda.synchronize()
    dt2 = (time.perf_counter() - t0) / 50
    print(f"{mb} MB D2H pinned {dt*1e6:.1f} us ({mb*1e3/dt/1e6:.1f} GB/s)  pageable {dt2*1e6:.1f} us")
