"""Per-op-kind cycle breakdown of hps_leaf_kernel (clock64 counters, diagnostics build path)."""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2503_04033_b200.engine import LeafEngine, dtn_flops, dtn_flops_executed

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=16)
ap.add_argument("--leaves", type=int, default=296)
ap.add_argument("--mode", default="dtn")
a = ap.parse_args()
tpl, pack = bench.make_shard(a.p, 16, 40.0, 0, 1, a.leaves)
eng = LeafEngine(tpl, False, True)
coeffs = torch.from_numpy(pack).cuda()
f = torch.randn(a.leaves, eng.n, dtype=torch.float64, device="cuda")
def run():
    if a.mode == "dtn":
        eng.dtn(coeffs)
    else:
        eng.reduce_load(coeffs, f)
run(); torch.cuda.synchronize()
cnt = torch.zeros(eng.slots * 64, dtype=torch.int64, device="cuda")
eng.lib.hps_plan_set_profile(eng.plan, ctypes.c_void_p(cnt.data_ptr()))
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); run(); e1.record(); torch.cuda.synchronize()
eng.lib.hps_plan_set_profile(eng.plan, ctypes.c_void_p(0))
ms = e0.elapsed_time(e1)
c = cnt.view(eng.slots, 64).cpu().numpy().astype(float)
names = ["small-panel", "swaps", "inv-lower", "inv-upper", "gemm-sub", "gemm-set", "gemm-set-Q", "gemm-sub-abi", "copy-abb"]
tot = c[:, :9].sum() + c[:, 22].sum() + c[:, 23].sum() + c[:, 24].sum() + c[:, 27].sum()
leaves = c[:, 9].sum()
print(f"p={a.p} leaves={a.leaves} mode={a.mode} kernel {ms:.1f} ms, {a.leaves/ms*1e3:.1f} leaves/s, "
      f"{a.leaves*dtn_flops_executed(eng.n, eng.m, a.p-2)/ms/1e9:.2f} TFLOP/s executed, "
      f"{a.leaves*dtn_flops(eng.n, eng.m)/ms/1e9:.2f} reference-equivalent")
clk = 1.965e9
for i, nm in list(enumerate(names)) + [(24, "rhs-profile"), (27, "W-block io"), (22, "assemble"), (23, "output")]:
    if c[:, i].sum() == 0:
        continue
    print(f"  {nm:12s} {100*c[:, i].sum()/tot:6.2f}%   {c[:, i].sum()/leaves/clk*1e3:8.2f} ms/leaf")
for b, nm in enumerate(["N<=64", "N<=256", "N>256"]):
    cyc, mf = c[:, 16 + b].sum(), c[:, 19 + b].sum() * 2**20
    if cyc:
        print(f"    gemm {nm:7s} {cyc/leaves/clk*1e3:8.2f} ms/leaf  {mf/leaves:.2e} flop/leaf  "
              f"{mf/cyc*clk/1e9:6.1f} GF/s per CTA")
for i, nm in zip(range(10, 15), ["p1-utop", "p2-gather", "p3-pivot", "p4-writeback", "p5-swaps"]):
    print(f"    {nm:12s} {c[:, i].sum()/leaves/clk*1e3:8.2f} ms/leaf")
print("  phases (all ops): " + ", ".join(f"{nm} {c[:, 28 + i].sum()/leaves/clk*1e3:.1f} ms/leaf" for i, nm in enumerate(["LU", "forward solve", "W blocks / backward"])))
print(f"  trailing-update k ranges skipped (row first-nonzero): {c[:, 31].sum() * 2**20 / leaves:.3e} flop/leaf")
print(f"  endgame helper time per CTA (mean over CTAs): {c[:, 26].mean()/clk*1e3:.1f} ms")
print(f"  row interchanges per leaf: {c[:, 15].sum()/leaves:.0f} of {eng.n} pivots")
gf = sum(c[:, 19 + b].sum() for b in range(3)) * 2**20
print(f"  gemm flops/leaf {gf/leaves:.3e}; gemm-only rate per CTA {gf/(c[:, 16:19].sum())*clk/1e9:.1f} GFLOP/s "
      f"(peak 251/SM); per-leaf total {tot/leaves/clk*1e3:.1f} ms")
# per-CTA spread (one leaf per CTA when leaves == slots): busy cycles by SM id
busy = c[:, :9].sum(1) + c[:, 22] + c[:, 23] + c[:, 24] + c[:, 27]
per_leaf = busy / np.maximum(c[:, 9], 1)
sm = c[:, 25].astype(int)
q = np.quantile(per_leaf, [0, 0.1, 0.5, 0.9, 1.0]) / clk * 1e3
print("  per-CTA ms/leaf quantiles (0,10,50,90,100%):", " ".join(f"{x:.1f}" for x in q))
lo = per_leaf[sm < sm.max() / 2].mean() / clk * 1e3
hi = per_leaf[sm >= sm.max() / 2].mean() / clk * 1e3
print(f"  mean ms/leaf on SM ids < half: {lo:.1f}, >= half: {hi:.1f}")
order = np.argsort(sm)
pair = per_leaf[order].reshape(-1, 2) if len(order) % 2 == 0 else None
if pair is not None:
    print(f"  same-SM pair |difference| mean {np.abs(pair[:, 0] - pair[:, 1]).mean() / clk * 1e3:.1f} ms")
ex = c[:, 32:35].sum()
if ex > 0:   # HPS_PROF_EXEC build: DMMA flops actually issued
    print(f"  executed DMMA flops/leaf {ex/leaves:.3e}")
    for b, nm in enumerate(["N<=64", "N<=256", "N>256"]):
        cyc, f = c[:, 16 + b].sum(), c[:, 32 + b].sum()
        if cyc:
            cap = c[:, 41 + b].sum()
            print(f"    gemm {nm:7s} executed {f/leaves:.2e} flop/leaf  {f/cyc*clk/1e9:6.1f} GF/s per CTA "
                  f"({100*f/cyc*clk/1e9/125.3:.0f}% of the 37.1/296 fair share); warp-slot use "
                  f"{100*f/max(cap, 1):.0f}% of the chunks walked, walked-chunk rate "
                  f"{cap/cyc*clk/1e9:6.1f} GF/s per CTA")
    for i, nm in enumerate(["LU", "forward solve", "W blocks / backward"]):
        cyc, f = c[:, 38 + i].sum(), c[:, 35 + i].sum()
        if cyc:
            print(f"    phase {nm:20s} gemm {cyc/leaves/clk*1e3:7.2f} ms/leaf, executed {f/leaves:.2e} flop/leaf, "
                  f"{f/cyc*clk/1e9:6.1f} GF/s per CTA; whole phase {c[:, 28 + i].sum()/leaves/clk*1e3:.1f} ms/leaf")
if c[:, 57:60].sum() > 0:   # HPS_PROF_GEMM build: where thread 0's GEMM time goes
    print("  GEMM time of thread 0 by N bucket (ms/leaf): setup | producer (of which: waiting for a released stage)"
          " | stage-data waits | tail; chunks/leaf")
    for b, nm in enumerate(["N<=64", "N<=256", "N>256"]):
        f = lambda k: c[:, k + b].sum() / leaves / clk * 1e3
        print(f"    {nm:7s} {f(48):7.2f} | {f(60):7.2f} ({f(44):7.2f}) | {f(51):7.2f} | {f(54):7.2f};"
              f"  {c[:, 57 + b].sum() / leaves:8.0f}")
    f = lambda k: c[:, k].sum() / leaves / clk * 1e3
    print(f"    producer, all buckets: tile claim + k bounds {f(47):.2f} ms/leaf, chunk issue (expect_tx, TMA, prefetch) {f(63):.2f} ms/leaf")
if c[:, 44:48].sum() > 0 and c[:, 57:60].sum() == 0:   # HPS_PROF_PIVOT build
    f = lambda k: c[:, k].sum() / leaves / clk * 1e3
    print(f"  pivot columns (thread 0, ms/leaf): selection + bookkeeping + 1/pivot {f(44):.2f}, row updates {f(45):.2f},"
          f" warp argmax + stash {f(46):.2f}, column barrier {f(47):.2f}")
