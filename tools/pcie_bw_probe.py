"""Host <-> device copy bandwidth from pinned memory (the e2e path's copies): 25 MB (x) and
67 MB (x, v, m, u) each way, CUDA events around torch copies.
  python tools/pcie_bw_probe.py"""
import torch, time
for mb in (25.2, 67):
    n = int(mb * 1e6 / 4)
    h = torch.empty(n).pin_memory(); d = torch.empty(n, device="cuda")
    for it in range(3):
        torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); d.copy_(h, non_blocking=True); e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        e0.record(); h.copy_(d, non_blocking=True); e1.record(); torch.cuda.synchronize()
        t2 = e0.elapsed_time(e1)
        print(f"{mb} MB H2D {t:.3f} ms {mb/t:.1f} GB/s  D2H {t2:.3f} ms {mb/t2:.1f} GB/s")
