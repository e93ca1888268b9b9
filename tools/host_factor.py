"""configs[4], second half: leaf reduction (GPU) vs host block-sparse assembly and
sparse factorization, per polynomial order, through the public solver API.

For each p the mesh is a g^3 leaf cube with g = round(N^(1/3) / p), so every row
has ~N DOFs (default N = 2.6e5: the largest size at which SuperLU factors the
p = 6 interface system in well under a minute on the host).  `condensation.build`
reports its own wall times: `dtn_assembly` (GPU leaf reduction through the
host-buffer C entry, incl. coefficient packing and the copies), `t_assembly`
(host scatter of DtN blocks into the block-sparse interface matrix) and
`factorize` (SuperLU, host).  One JSON row per p.
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2503_04033_b200 import build_discretization, MeshConfig, make_problem, solve_bvp
from paper_2503_04033_b200.engine import LeafEngine

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=float, default=2.6e5)
ap.add_argument("--ps", default="6,8,10,12,14,16,18,20,22")
ap.add_argument("--kappa", type=float, default=40.0)
a = ap.parse_args()
for p in (int(x) for x in a.ps.split(",")):
    g = max(2, int(round(a.N ** (1.0 / 3.0) / p)))
    spec = make_problem("bump_helmholtz", d=3, kappa=a.kappa)
    disc = build_discretization(spec.domain, MeshConfig((g, g, g), p))
    tic = time.perf_counter()
    report, sys_ = solve_bvp(disc, spec.coeffs, spec.f, spec.g)
    wall = time.perf_counter() - tic
    t = report.wall_times
    row = {"p": p, "leaf_grid": [g, g, g], "leaves": g ** 3, "dofs": int(disc.n_total),
           "interface_unknowns": int(sys_.n), "t_nnz": int(sys_.t.nnz),
           "leaf_reduction_s": t["dtn_assembly"], "t_assembly_s": t["t_assembly"],
           "factorize_s": t["factorize"], "load_reduction_s": t["load_reduction"],
           "interface_solve_s": t["interface_solve"], "interior_solve_s": t["interior_solve"],
           "solve_bvp_wall_s": wall, "residual": report.residual}
    print(json.dumps(row), flush=True)
    del sys_, report
    LeafEngine.clear_cache()
