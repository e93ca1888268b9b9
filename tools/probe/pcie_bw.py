"""Host<->device copy bandwidth with pinned buffers (context for the e2e number)."""
import time, torch
for gb in (1, 4):
    n = gb * (1 << 30) // 8
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 3
        print(f"{name} {gb} GiB pinned: {gb * 1.0737 / dt:.1f} GB/s")
