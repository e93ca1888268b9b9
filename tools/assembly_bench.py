"""Interface assembly: device scatter (assembly.py) vs the reference's host
scatter (HPS_HOST_ASSEMBLY=1) inside condensation.build, factorization
skipped.  Prints one JSON line per p: leaf-stage seconds, T assembly seconds,
T nnz, and whether both paths give bit-identical T and coupling."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2503_04033_b200 import MeshConfig, build_discretization, make_problem
from paper_2503_04033_b200 import condensation, sparse_backend

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=float, default=1e6)
ap.add_argument("--ps", default="8,12,16")
ap.add_argument("--kappa", type=float, default=40.0)
a = ap.parse_args()
sparse_backend_factor = sparse_backend.analyze_and_factor
condensation.sparse_backend.analyze_and_factor = lambda t: None   # leaf stage + assembly only


def run(disc, spec, host):
    os.environ["HPS_HOST_ASSEMBLY"] = "1" if host else "0"
    tic = time.perf_counter()
    s = condensation.build(disc, spec.coeffs)
    return s, time.perf_counter() - tic


for p in (int(x) for x in a.ps.split(",")):
    g = max(2, int(round(a.N ** (1.0 / 3.0) / p)))
    spec = make_problem("bump_helmholtz", d=3, kappa=a.kappa)
    disc = build_discretization(spec.domain, MeshConfig((g, g, g), p))
    run(disc, spec, False)  # plan creation, allocator warm-up
    hs, hw = run(disc, spec, True)
    ds, dw = run(disc, spec, False)
    same = all(np.array_equal(getattr(x, f), getattr(y, f))
               for x, y in ((hs.t, ds.t), (hs.dirichlet_coupling, ds.dirichlet_coupling))
               for f in ("indptr", "indices", "data"))
    print(json.dumps({"p": p, "leaves": g ** 3, "t_nnz": int(ds.t.nnz), "c_nnz": int(ds.dirichlet_coupling.nnz),
                      "host": {"leaf_stage_s": hs.build_times["dtn_assembly"], "t_assembly_s": hs.build_times["t_assembly"], "wall_s": hw},
                      "device": {"leaf_stage_s": ds.build_times["dtn_assembly"], "t_assembly_s": ds.build_times["t_assembly"], "wall_s": dw},
                      "bit_identical": bool(same)}), flush=True)
    del hs, ds
