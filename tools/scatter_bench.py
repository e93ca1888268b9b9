"""hps_interface_scatter on its own: device DtN maps of one flush (random
values, the mesh's real pattern and jobs) added into T and C, CUDA events on
the launching stream.  Algorithmic bytes per launch = 8 per scattered map
element (read) + 16 per CSR value of T and C (read-modify-write; the second
contribution to an entry of T meets it in L2); reported against the measured
HBM copy bandwidth in MEASURED_PEAKS.json."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2503_04033_b200 import MeshConfig, build_discretization, make_problem
from paper_2503_04033_b200.assembly import DeviceAssembler, InterfacePattern

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=16)
ap.add_argument("--g", type=int, default=6)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
spec = make_problem("bump_helmholtz", d=3, kappa=40.0)
disc = build_discretization(spec.domain, MeshConfig((a.g,) * 3, a.p))
pat = InterfacePattern(disc)
ids = list(range(len(disc.leaves)))
m = len(disc.leaves[0].boundary_ids)
dtn = torch.randn(len(ids), m, m, dtype=torch.float64, device="cuda")
asm = DeviceAssembler(pat, 0)
jobs = pat.jobs_for(ids)
elems = int((jobs[:, 3] * jobs[:, 4]).sum())
for _ in range(3):
    asm.add(dtn, ids)
torch.cuda.synchronize()
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(a.iters):
    e0.record(s)
    asm.add(dtn, ids)  # includes the jobs H2D (small) and one kernel
    e1.record(s)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e-3)
t = float(np.median(ts))
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 7700.0
alg = elems * 8 + 16 * (pat.nnz[0] + pat.nnz[1])
gbs = alg / t / 1e9
print(json.dumps({"kernel": "hps_interface_scatter_kernel", "p": a.p, "leaves": len(ids), "jobs": int(len(jobs)),
                  "elements": elems, "t_nnz": pat.nnz[0], "c_nnz": pat.nnz[1], "s_per_launch": t,
                  "algorithmic_bytes": alg, "achieved_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak}))
