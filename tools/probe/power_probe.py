"""Board power and SM clock under three sustained loads (8 s each), nvidia-smi sampled:
cuBLAS DGEMM (DMMA-bound, L2-resident), an HBM copy stream, and the leaf kernel
(p = 16, 4096 leaves).  Shows which activity drives the 1 kW cap the leaf kernel hits."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402


def sustained(fn, seconds, work):
    fn()
    torch.cuda.synchronize()
    with bench.ClockSampler(0) as clk:
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        t0 = time.time()
        e0.record()
        k = 0
        while time.time() - t0 < seconds:
            fn()
            k += 1
            if k % 4 == 0:
                torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    summ = clk.summary()
    pw = []
    try:
        for line in open(clk.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7 and parts[2].replace(".", "").isdigit():
                pw.append(float(parts[2]))
    except OSError:
        pass
    summ["power_w_median"] = float(np.median(pw)) if pw else None
    return {"rate": work * k / (ms / 1e3), "calls": k, "seconds": ms / 1e3, "clocks": summ}


out = {}
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
r = sustained(lambda: a @ b, 8.0, 2.0 * n ** 3)
out["dgemm_8192"] = dict(r, rate_tflops=r["rate"] / 1e12)
del a, b
x = torch.empty(2 ** 30, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
r = sustained(lambda: y.copy_(x), 8.0, 2 * x.numel() * 8)
out["hbm_copy_8GB"] = dict(r, rate_gbs=r["rate"] / 1e9)
del x, y
torch.cuda.empty_cache()
from paper_2503_04033_b200.engine import LeafEngine, dtn_flops_executed  # noqa: E402
tpl, pack = bench.make_shard(16, 16, 40.0)
eng = LeafEngine(tpl, False, True)
coeffs = torch.from_numpy(pack).cuda()
m = tpl.n_boundary
o = torch.empty((pack.shape[0], m, m), dtype=torch.float64, device="cuda")
st = torch.empty((pack.shape[0], 2), dtype=torch.float64, device="cuda")
r = sustained(lambda: eng.dtn(coeffs, o, st), 12.0, pack.shape[0])
out["leaf_kernel_p16"] = dict(r, maps_per_s=r["rate"],
                              tflops_executed=r["rate"] * dtn_flops_executed(tpl.n_interior, m, 14) / 1e12)
print(json.dumps(out, indent=1))
