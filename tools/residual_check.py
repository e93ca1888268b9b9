"""solve_bvp residual / interface RHS norm through both assembly paths (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2503_04033_b200 import MeshConfig, build_discretization, make_problem, solve_bvp
from paper_2503_04033_b200.condensation import reduce_load, build
spec = make_problem("bump_helmholtz", d=3, kappa=40.0)
disc = build_discretization(spec.domain, MeshConfig((4, 4, 4), 8))
for host in ("1", "0"):
    os.environ["HPS_HOST_ASSEMBLY"] = host
    report, s = solve_bvp(disc, spec.coeffs, spec.f, spec.g)
    v, g_b = reduce_load(disc, spec.coeffs, spec.f, spec.g, s)
    r = s.t @ report.u[disc.index_interface] - g_b
    print("host" if host == "1" else "device", "residual", report.residual, "|g_b|", np.linalg.norm(g_b),
          "|T u - g|", np.linalg.norm(r), "|T|", abs(s.t).sum(), "|u|", np.linalg.norm(report.u))
