"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container only (needs /root/reference, which does not exist
on the GPU box):

    python tests/golden/make_golden.py [leaf] [pipeline] [bench]   (default: all)

For every case it imports ``steklov`` from /root/reference/pkg/src, builds the
leaf template and operator with the reference's own code, and stores inputs
(coefficients sampled at interior nodes, exactly the arrays the reference
evaluates) and outputs (A_ii, A_ib, a_bi, a_bb, DtN, S, reduced load, interior
solve) in ``leaf_cases.npz``.  A second file, ``pipeline_cases.npz``, stores
end-to-end ``solve_bvp`` results and assembled interface matrices for small
meshes.  ``bench_cases.npz`` holds the reference's leaf outputs at the
benchmark orders (configs[1-3]: p = 12, 16, 20; probes and sampled rows of the
maps, full vectors).  The fixtures are what pin the oracle
(tests/test_oracle_golden.py) and the CUDA path (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from steklov import condensation as ref_cond  # noqa: E402
from steklov.geometry import DomainBox, MeshConfig, build_discretization  # noqa: E402
from steklov.geometry import sinusoidal_map  # noqa: E402
from steklov.local_ops import (CoefficientField, LeafTemplate,  # noqa: E402
                               build_leaf_factors, cheb_nodes, isotropic_field)
from steklov.problems import make_problem  # noqa: E402


def bump(x, kappa):
    c = np.full(x.shape[1], 0.5)
    r2 = ((x - c[None, :]) ** 2).sum(axis=1)
    return -kappa * kappa * (1.0 - 0.5 * np.exp(-r2 / (2 * 0.15 ** 2)))


LEAF_CASES = [
    # name, d, p, lo, hi, field kind
    ("lap2_p6", 2, 6, (0.0, 0.0), (1.0, 1.0), "laplace"),
    ("helm2_p7", 2, 7, (0.0, 0.5), (0.5, 1.0), "helm_const"),
    ("conv2_p8", 2, 8, (-0.5, -0.5), (0.0, 0.0), "convdiff"),
    ("lap3_p5", 3, 5, (0.0, 0.0, 0.0), (0.5, 0.5, 0.5), "laplace"),
    ("bump3_p6", 3, 6, (0.25, 0.5, 0.0), (0.5, 0.75, 0.25), "bump"),
    ("grav3_p8", 3, 8, (1.1, -1.0, -1.2), (1.35, -0.75, -0.95), "gravity"),
    ("conv3_p7", 3, 7, (-0.5, -0.5, 0.0), (0.0, 0.0, 0.5), "convdiff"),
    ("bump3_p10", 3, 10, (0.375, 0.375, 0.375), (0.5, 0.5, 0.5), "bump"),
    # legendre face grids (corner_mode="legendre"), with and without cross terms
    ("leg_curv2_p6", 2, 6, (1.1, -1.0), (1.6, -0.5), "curved"),
    ("leg_curv3_p5", 3, 5, (1.1, -1.0, -1.2), (1.6, -0.5, -0.7), "curved"),
    ("leg_curv3_p7", 3, 7, (1.35, -0.75, -0.95), (1.6, -0.5, -0.7), "curved"),
    ("leg_lap3_p6", 3, 6, (0.0, 0.0, 0.0), (0.5, 0.5, 0.5), "laplace"),
    ("leg_grav2_p8", 2, 8, (1.1, -1.0), (1.35, -0.75), "gravity"),
]


def field(kind, d):
    if kind == "laplace":
        return isotropic_field(d)
    if kind == "helm_const":
        return isotropic_field(d, zeroth=lambda x: np.full(x.shape[0], -81.0))
    if kind == "bump":
        return isotropic_field(d, zeroth=lambda x: bump(x, 12.0))
    if kind == "gravity":
        return isotropic_field(d, zeroth=lambda x: -144.0 * (1.0 - x[:, d - 1]))
    if kind == "curved":
        base = isotropic_field(d, zeroth=lambda x: np.full(x.shape[0], -36.0))
        return sinusoidal_map(0.25, 6.0).coefficient_transform(base)
    if kind == "convdiff":
        def first(x):
            b = np.zeros_like(x)
            b[:, 0] = -np.cos(x[:, 0]) * np.sin(x[:, 1])
            b[:, 1] = np.sin(x[:, 0]) * np.cos(x[:, 1])
            return 0.025 * b
        return isotropic_field(d, diffusion=0.3,
                               zeroth=lambda x: 1.0 + 0.1 * x[:, 0], first=first)
    raise ValueError(kind)


def pack_coeffs(coeffs, x_int, d):
    """(ncoef, n): diag second order, cross sums a_ab + a_ba (if has_cross_terms),
    first order (if any), zeroth (if any)."""
    a2 = np.asarray(coeffs.second_order(x_int), dtype=float)
    rows = [a2[:, k, k] for k in range(d)]
    if coeffs.has_cross_terms:
        rows += [a2[:, a, b] + a2[:, b, a] for a in range(d) for b in range(a + 1, d)]
    if coeffs.first_order is not None:
        a1 = np.asarray(coeffs.first_order(x_int), dtype=float)
        rows += [a1[:, k] for k in range(d)]
    if coeffs.zeroth_order is not None:
        rows.append(np.asarray(coeffs.zeroth_order(x_int), dtype=float))
    return np.stack(rows)


def leaf_cases():
    out = {}
    rng = np.random.default_rng(20250305)
    for name, d, p, lo, hi, kind in LEAF_CASES:
        lo, hi = np.asarray(lo), np.asarray(hi)
        widths = hi - lo
        mode = "legendre" if name.startswith("leg_") else "drop"
        coeffs = field(kind, d)
        tpl = LeafTemplate(widths, p, mode, coeffs.has_cross_terms)
        nodes = []
        for k in range(d):
            x = lo[k] + widths[k] * tpl.ref_offsets
            x[0], x[-1] = lo[k], hi[k]
            nodes.append(x)
        grid = tpl.leaf_grid(nodes)
        lf = build_leaf_factors(tpl, coeffs, grid, leaf_index=(0,) * d)
        a_ii, a_ib = tpl.interior_blocks(coeffs, grid)
        x_int = grid[tpl.interior_idx]
        f = np.sin(3 * x_int[:, 0]) + x_int[:, -1] ** 2
        v = lf.solve_interior(f)
        ub = rng.standard_normal(tpl.n_boundary)
        u_int = v - lf.solve_interior(a_ib @ ub)
        pre = name + "/"
        out[pre + "meta"] = np.array([d, p, 1 if coeffs.first_order is not None else 0,
                                      1 if coeffs.zeroth_order is not None else 0,
                                      1 if mode == "legendre" else 0,
                                      1 if coeffs.has_cross_terms else 0])
        out[pre + "widths"] = widths
        out[pre + "coeffs"] = pack_coeffs(coeffs, x_int, d)
        out[pre + "a_ii"] = a_ii
        out[pre + "a_ib"] = a_ib
        out[pre + "a_bi"] = tpl.a_bi
        out[pre + "a_bb"] = tpl.a_bb
        out[pre + "dtn"] = lf.dtn
        out[pre + "s"] = lf.s
        out[pre + "f"] = f
        out[pre + "v"] = v
        out[pre + "flux"] = tpl.a_bi @ v
        out[pre + "ub"] = ub
        out[pre + "u_int"] = u_int
        out[pre + "interior_idx"] = tpl.interior_idx
        if mode == "drop":
            out[pre + "bcols"] = tpl._bcols
        else:
            out[pre + "Q"] = tpl._boundary_injection
        out[pre + "D"] = np.stack(tpl.diff)
    return out


PIPELINE_CASES = [
    # name, problem, d, params, boxes, p
    ("poisson2_2x2_p6", "poisson_green", 2, {}, (2, 2), 6),
    ("gravity2_3x2_p7", "gravity_helmholtz", 2, {"kappa": 5.0}, (3, 2), 7),
    ("helm3_2x2x2_p6", "helmholtz_green", 3, {"kappa": 6.0}, (2, 2, 2), 6),
    ("convdiff3_2x1x2_p5", "convdiff_step", 3, {}, (2, 1, 2), 5),
    ("curved2_2x2_p6_leg", "curved_helmholtz", 2, {"kappa": 4.0}, (2, 2), 6),
    ("curved3_2x1x1_p5_leg", "curved_helmholtz", 3, {"kappa": 4.0}, (2, 1, 1), 5),
    # BASELINE configs[0]: 3D Poisson, p = 8, 2x2x2 leaves, manufactured (Green's function) solution
    ("poisson3_2x2x2_p8", "poisson_green", 3, {}, (2, 2, 2), 8),
]


def pipeline_cases():
    out = {}
    for name, prob_name, d, params, boxes, p in PIPELINE_CASES:
        prob = make_problem(prob_name, d=d, **params)
        mode = "legendre" if name.endswith("_leg") else "drop"
        disc = build_discretization(prob.domain, MeshConfig(boxes, p, mode))
        report, sys_ = ref_cond.solve_bvp(disc, prob.coeffs, prob.f, prob.g)
        pre = name + "/"
        out[pre + "u"] = report.u
        out[pre + "nodes"] = disc.nodes
        out[pre + "t_dense"] = sys_.t.toarray()
        out[pre + "residual"] = np.array([report.residual])
        if prob.exact is not None:
            out[pre + "exact"] = prob.exact(disc.nodes)
    return out


def bench_field(kind, kappa):
    """The bench workloads' coefficient fields (bench.py make_shard):
    -Lap u - kappa^2 b(x) u with the Gaussian bump, or b = 1."""
    if kind == "const":
        return isotropic_field(3, zeroth=lambda x: np.full(x.shape[0], -kappa * kappa))
    return isotropic_field(3, zeroth=lambda x: bump(x, kappa))


BENCH_CASES = [
    # name, p, leaf boxes per axis, kappa, field, leaf indices (i, j, k) in the unit-cube grid
    # configs[1]: constant coefficient, every leaf the same operator up to translation
    ("c1_p12_const_k10", 12, 8, 10.0, "const", [(3, 4, 5)]),
    # configs[2]: (7,7,7) has the bump centre (0.5, 0.5, 0.5) as its corner; (3,12,5) off-centre
    ("c2_p16_bump_k40", 16, 16, 40.0, "bump", [(7, 7, 7), (3, 12, 5)]),
    # configs[3]: (1,7,7) is in rank 0's 1/8 share (leaves 0-511) nearest the centre
    ("c3_p20_bump_k80", 20, 16, 80.0, "bump", [(7, 7, 7), (1, 7, 7)]),
]
N_PROBE = 8     # random probe columns for the DtN map and the solution operator
N_ROWS = 8      # full DtN rows stored per leaf


def bench_cases():
    """Reference outputs at the benchmark orders (p = 12, 16, 20).  Full m x m maps
    would be 3-30 MB each, so the fixtures keep what pins them: T R and S R for a
    seeded Gaussian probe R (m x 8), N_ROWS full rows of T, the Frobenius norms,
    and the full vectors of the load reduction and the interior solve
    (reference local_ops.py:439-446, condensation.py:314-323 and 372-383)."""
    out = {}
    rng = np.random.default_rng(20251019)
    for name, p, boxes, kappa, kind, leaves in BENCH_CASES:
        h = 1.0 / boxes
        coeffs = bench_field(kind, kappa)
        tpl = LeafTemplate(np.array([h, h, h]), p, "drop", False)
        m, n = tpl.n_boundary, tpl.n_interior
        R = rng.standard_normal((m, N_PROBE))
        out[name + "/meta"] = np.array([p, boxes, kappa])
        out[name + "/R"] = R
        for idx in leaves:
            lo = np.asarray(idx, dtype=float) * h
            nodes = []
            for k in range(3):
                x = lo[k] + h * tpl.ref_offsets
                x[0], x[-1] = lo[k], lo[k] + h
                nodes.append(x)
            grid = tpl.leaf_grid(nodes)
            lf = build_leaf_factors(tpl, coeffs, grid, leaf_index=idx)
            a_ii, a_ib = tpl.interior_blocks(coeffs, grid)
            x_int = grid[tpl.interior_idx]
            f = np.sin(3 * x_int[:, 0]) + x_int[:, -1] ** 2
            v = lf.solve_interior(f)
            ub = rng.standard_normal(m)
            u_int = v - lf.solve_interior(a_ib @ ub)
            rows = np.sort(rng.choice(m, N_ROWS, replace=False))
            pre = f"{name}/{idx[0]}_{idx[1]}_{idx[2]}/"
            out[pre + "coeffs"] = pack_coeffs(coeffs, x_int, 3)
            out[pre + "dtn_R"] = lf.dtn @ R
            out[pre + "dtn_rows_idx"] = rows
            out[pre + "dtn_rows"] = lf.dtn[rows]
            out[pre + "dtn_fro"] = np.array([np.linalg.norm(lf.dtn)])
            out[pre + "s_R"] = lf.s @ R
            out[pre + "s_fro"] = np.array([np.linalg.norm(lf.s)])
            out[pre + "f"] = f
            out[pre + "v"] = v
            out[pre + "flux"] = tpl.a_bi @ v
            out[pre + "ub"] = ub
            out[pre + "u_int"] = u_int
            diag = np.abs(np.diag(lf.a_ii_factor[0]))
            out[pre + "pivots"] = np.array([diag.min(), diag.max(),
                                            int((lf.a_ii_factor[1] != np.arange(n)).sum())])
    return out


def main():
    only = sys.argv[1:]
    if not only or "leaf" in only:
        np.savez_compressed(os.path.join(HERE, "leaf_cases.npz"), **leaf_cases())
    if not only or "pipeline" in only:
        np.savez_compressed(os.path.join(HERE, "pipeline_cases.npz"), **pipeline_cases())
    if not only or "bench" in only:
        np.savez_compressed(os.path.join(HERE, "bench_cases.npz"), **bench_cases())
    for fn in ("leaf_cases.npz", "pipeline_cases.npz", "bench_cases.npz"):
        print(fn, os.path.getsize(os.path.join(HERE, fn)), "bytes")


if __name__ == "__main__":
    main()
