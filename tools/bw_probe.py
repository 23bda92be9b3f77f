import torch, time
n = 25 * 1024 * 1024 // 4 * 4
a = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for k in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d.copy_(a, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter()
    a.copy_(d, non_blocking=True); torch.cuda.synchronize()
    t2 = time.perf_counter()
    print("H2D %.1f GB/s  D2H %.1f GB/s" % (n*4/(t1-t0)/1e9, n*4/(t2-t1)/1e9))
