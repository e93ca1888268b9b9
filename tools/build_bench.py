"""Throughput of the drop-in build() leaf stage against the bare LeafEngine bench.

  python tools/build_bench.py --boxes 16 --p 16 --flushes 592,1184,2048,4096 [--assemble]

For each flush size (leaves per launch, set through BatchSchedule.memory_budget =
flush x staged-map bytes) it runs condensation.build() on the bump Helmholtz
problem (kappa = 40, the bench's coefficients) and reports the leaf stage
(coefficient evaluation + packing on the host, pinned H2D, one kernel launch per
flush, the scatter into T on the same stream, the pivot check) next to
LeafEngine.dtn on the same leaves with the coefficients already in HBM.  The
sparse factorization is excluded (monkeypatched out).  Without --assemble the
scatter into T is skipped as well: at 16^3 leaves and p = 16, T would hold
~4.9e9 nonzeros, far beyond what the host side (pattern, SuperLU) can take.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402
import torch  # noqa: E402

from paper_2503_04033_b200 import condensation, sparse_backend  # noqa: E402
from paper_2503_04033_b200.engine import LeafEngine  # noqa: E402
from paper_2503_04033_b200.geometry import MeshConfig, build_discretization  # noqa: E402
from paper_2503_04033_b200.problems import make_problem  # noqa: E402


class NullAssembler:
    """Stands in for DeviceAssembler when T is not assembled (scatter skipped)."""

    def __init__(self, pattern, device, vectors=False):
        self.t_vals = self.c_vals = torch.zeros(1, dtype=torch.float64)

    def add(self, dtn, ids):
        pass

    def finish(self):
        return sp.identity(1, format="csr"), sp.csr_matrix((1, 1))


class NullPattern:
    nnz = (1, 1)


ap = argparse.ArgumentParser()
ap.add_argument("--boxes", type=int, default=16)
ap.add_argument("--p", type=int, default=16)
ap.add_argument("--kappa", type=float, default=40.0)
ap.add_argument("--flushes", default="592,1184,2048,4096")
ap.add_argument("--assemble", action="store_true")
a = ap.parse_args()

spec = make_problem("bump_helmholtz", d=3, kappa=a.kappa)
t0 = time.perf_counter()
disc = build_discretization(spec.domain, MeshConfig((a.boxes,) * 3, a.p))
geo_s = time.perf_counter() - t0
L = len(disc.leaves)
sparse_backend_factor = sparse_backend.analyze_and_factor
condensation.sparse_backend.analyze_and_factor = lambda t: None   # factorization excluded
if not a.assemble:
    condensation.DeviceAssembler = NullAssembler
    condensation.pattern_for = lambda disc: NullPattern()

# the bare engine on the same leaves (coefficients in HBM, CUDA events)
from paper_2503_04033_b200.local_ops import LeafTemplate, pack_coefficients  # noqa: E402
tpl = LeafTemplate(disc.leaf_widths, a.p, disc.corner_mode, False)
t0 = time.perf_counter()
pack = pack_coefficients(spec.coeffs, condensation.interior_points(disc, range(L)), L)
pack_s = time.perf_counter() - t0
eng = LeafEngine.for_template(tpl, spec.coeffs)
coeffs = torch.from_numpy(pack).cuda()
out = torch.empty((L, tpl.n_boundary, tpl.n_boundary), dtype=torch.float64, device="cuda")
stats = torch.empty((L, 2), dtype=torch.float64, device="cuda")
eng.dtn(coeffs, out, stats)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
eng.dtn(coeffs, out, stats)
e1.record()
torch.cuda.synchronize()
engine_s = e0.elapsed_time(e1) / 1e3
del out, coeffs, stats
torch.cuda.empty_cache()
print(json.dumps({"what": "engine", "leaves": L, "p": a.p, "seconds": engine_s, "leaves_per_s": L / engine_s,
                  "host_pack_all_s": pack_s, "geometry_s": geo_s}), flush=True)

block = 8 * tpl.n_boundary ** 2
for flush in (int(x) for x in a.flushes.split(",")):
    sched = condensation.BatchSchedule(memory_budget=flush * block + block // 2)
    for rep in range(2):
        t0 = time.perf_counter()
        sys_ = condensation.build(disc, spec.coeffs, sched)
        wall = time.perf_counter() - t0
        bt = sys_.build_times
        print(json.dumps({"what": "build", "rep": rep, "flush": flush, "leaves": L, "p": a.p,
                          "assemble_T": a.assemble, "leaf_stage_s": bt["dtn_assembly"],
                          "t_assembly_s": bt["t_assembly"], "wall_s": wall,
                          "leaf_stage_leaves_per_s": L / bt["dtn_assembly"],
                          "vs_engine": engine_s / bt["dtn_assembly"],
                          "peak_staged_bytes": sys_.peak_workspace_bytes,
                          "device_workspace_bytes": sys_.device_workspace_bytes}), flush=True)
        del sys_
