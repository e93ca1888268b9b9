"""configs[4]: polynomial-order sweep of the GPU leaf reduction at fixed N ~ 1e7 DOFs.

For each p, the number of leaves is N / p^3 (rounded); the kernel time is the
device-resident DtN batch (inputs in HBM, CUDA events), i.e. the leaf-reduction
part of the build stage.  The host sparse factorization at this N is out of reach
for SuperLU on the host and is reported separately at smaller N (tools/host_factor.py).
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2503_04033_b200.engine import LeafEngine, dtn_flops, dtn_flops_executed

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=float, default=1e7)
ap.add_argument("--ps", default="6,8,10,12,14,16,18,20,22")
ap.add_argument("--max-leaves", type=int, default=0)
a = ap.parse_args()
rows = []
for p in (int(x) for x in a.ps.split(",")):
    L = int(round(a.N / p ** 3))
    if a.max_leaves:
        L = min(L, a.max_leaves)
    tpl, pack = bench.make_shard(p, 16, 40.0, 0, 1, L)
    eng = LeafEngine(tpl, False, True)
    coeffs = torch.from_numpy(pack).cuda()
    n, m = eng.n, eng.m
    out = torch.empty((L, m, m), dtype=torch.float64, device="cuda")
    stats = torch.empty((L, 2), dtype=torch.float64, device="cuda")
    # untimed launches until ~1 s of work: the first order of the sweep otherwise
    # runs before the SM clocks have ramped up
    import time
    t_w = time.perf_counter()
    while True:
        eng.dtn(coeffs, out, stats)
        torch.cuda.synchronize()
        if time.perf_counter() - t_w > 1.0:
            break
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); eng.dtn(coeffs, out, stats); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    row = {"p": p, "leaves": L, "dofs": L * p ** 3, "slots": eng.slots, "seconds": ms / 1e3,
           "leaves_per_s": L / ms * 1e3,
           "tflops_executed": L * dtn_flops_executed(n, m, p - 2) / ms / 1e9,
           "tflops_reference_equivalent": L * dtn_flops(n, m) / ms / 1e9}
    print(json.dumps(row), flush=True)
    rows.append(row)
    del out, coeffs, stats, eng
    LeafEngine.clear_cache()
    torch.cuda.empty_cache()
