"""Library FP64 context numbers on B200: cuBLAS DGEMM and cuSOLVER getrf via torch."""
import time, torch
dev = "cuda:0"
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
for n in (2048, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=dev); b = torch.randn(n, n, dtype=torch.float64, device=dev)
    ms = timeit(lambda: a @ b)
    print(f"cuBLAS DGEMM n={n}: {2*n**3/ms/1e9:.2f} TFLOP/s ({ms:.2f} ms)")
# sustained DGEMM ~4s
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device=dev); b = torch.randn(n, n, dtype=torch.float64, device=dev)
torch.cuda.synchronize(); t0 = time.time(); k = 0
e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True); e0.record()
while time.time() - t0 < 4.0:
    c = a @ b; k += 1
    if k % 4 == 0: torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
print(f"cuBLAS DGEMM sustained n={n}: {2*n**3*k/e0.elapsed_time(e1)/1e9:.2f} TFLOP/s over {k} calls")
for n, bs in ((216, 512), (1000, 64), (2744, 8), (5832, 2)):
    a = torch.randn(bs, n, n, dtype=torch.float64, device=dev) + n * torch.eye(n, dtype=torch.float64, device=dev)
    ms = timeit(lambda: torch.linalg.lu_factor(a), reps=3)
    print(f"torch lu_factor batch={bs} n={n}: {bs*2/3*n**3/ms/1e9:.3f} TFLOP/s ({ms:.2f} ms)")
