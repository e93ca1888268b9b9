"""Full two-level pipeline (GPU leaf work + host sparse solve) vs the reference.

The golden file holds the reference package's own solve_bvp outputs and
assembled interface matrices (tests/golden/make_golden.py).  Tolerance: 1e-10
relative (north star; reference acceptance criterion 1).
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
PG = np.load(os.path.join(HERE, "golden", "pipeline_cases.npz"))
CASES = [
    ("poisson2_2x2_p6", "poisson_green", 2, {}, (2, 2), 6),
    ("gravity2_3x2_p7", "gravity_helmholtz", 2, {"kappa": 5.0}, (3, 2), 7),
    ("helm3_2x2x2_p6", "helmholtz_green", 3, {"kappa": 6.0}, (2, 2, 2), 6),
    ("convdiff3_2x1x2_p5", "convdiff_step", 3, {}, (2, 1, 2), 5),
    ("curved2_2x2_p6_leg", "curved_helmholtz", 2, {"kappa": 4.0}, (2, 2), 6),
    ("curved3_2x1x1_p5_leg", "curved_helmholtz", 3, {"kappa": 4.0}, (2, 1, 1), 5),
    # BASELINE configs[0]: 3D Poisson, p = 8, 2x2x2 leaves, manufactured (Green's function) solution
    ("poisson3_2x2x2_p8", "poisson_green", 3, {}, (2, 2, 2), 8),
]


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def setup(prob, d, params, boxes, p, schedule=None, mode="drop"):
    from paper_2503_04033_b200 import build_discretization, MeshConfig, make_problem, solve_bvp
    spec = make_problem(prob, d=d, **params)
    disc = build_discretization(spec.domain, MeshConfig(boxes, p, mode))
    report, sys_ = solve_bvp(disc, spec.coeffs, spec.f, spec.g, schedule=schedule)
    return spec, disc, report, sys_


@pytest.mark.parametrize("name,prob,d,params,boxes,p", CASES)
def test_pipeline_matches_reference(name, prob, d, params, boxes, p):
    mode = "legendre" if name.endswith("_leg") else "drop"
    spec, disc, report, sys_ = setup(prob, d, params, boxes, p, mode=mode)
    assert rel(report.u, PG[name + "/u"]) <= 1e-10
    assert rel(sys_.t.toarray(), PG[name + "/t_dense"]) <= 1e-10
    assert report.residual <= 1e-10
    if name + "/exact" in PG.files:
        from paper_2503_04033_b200 import relative_l2_error
        ours = relative_l2_error(report.u, PG[name + "/exact"])
        theirs = relative_l2_error(PG[name + "/u"], PG[name + "/exact"])
        assert ours <= theirs * (1 + 1e-6) + 1e-14


def test_schedule_knobs_do_not_change_results():
    from paper_2503_04033_b200 import BatchSchedule
    a = setup("helmholtz_green", 3, {"kappa": 6.0}, (2, 2, 2), 6)[2].u
    b = setup("helmholtz_green", 3, {"kappa": 6.0}, (2, 2, 2), 6,
              BatchSchedule(batch_size=1, resident_limit=1, cache_leaf_factors=True))[2].u
    assert rel(a, b) <= 1e-13


def test_reuse_linearity_and_zero_data():
    from paper_2503_04033_b200 import run_solve_stage
    spec, disc, first, sys_ = setup("poisson_green", 2, {}, (2, 2), 6)
    zero = lambda x: np.zeros(x.shape[0])  # noqa: E731
    f1, g1 = (lambda x: np.sin(x[:, 0])), (lambda x: x[:, 0] * x[:, 1])
    f2, g2 = (lambda x: np.cos(x[:, 1])), (lambda x: x[:, 1] ** 2)
    u1 = run_solve_stage(sys_, f1, g1).u
    u2 = run_solve_stage(sys_, f2, g2)
    assert u2.wall_times["factorize"] == 0.0
    u12 = run_solve_stage(sys_, lambda x: 2 * f1(x) - f2(x), lambda x: 2 * g1(x) - g2(x)).u
    assert rel(u12, 2 * u1 - u2.u) <= 1e-12
    assert np.abs(run_solve_stage(sys_, zero, zero).u).max() == 0.0


def test_singular_leaf_reported():
    from paper_2503_04033_b200 import (CoefficientField, LeafSingularError, build,
                                       build_discretization, DomainBox, MeshConfig)
    coeffs = CoefficientField(second_order=lambda x: np.zeros((x.shape[0], 2, 2)),
                              zeroth_order=lambda x: np.zeros(x.shape[0]))
    disc = build_discretization(DomainBox((0.0, 0.0), (1.0, 1.0)), MeshConfig((2, 1), 5))
    with pytest.raises(LeafSingularError):
        build(disc, coeffs)


def test_build_leaf_operator_api():
    from paper_2503_04033_b200 import build_leaf_operator, laplace_field, cheb_nodes
    p = 6
    lf = build_leaf_operator(((0.0, 0.0), (1.0, 1.0)), p, laplace_field(2))
    assert np.abs(lf.dtn @ np.ones(lf.dtn.shape[1])).max() <= 1e-11 * np.abs(lf.dtn).max()
    xc = cheb_nodes(p, (0.0, 1.0))[1:-1]
    trace = np.concatenate([np.zeros(p - 2), np.ones(p - 2), xc, xc])
    expected = np.concatenate([-np.ones(p - 2), np.ones(p - 2), np.zeros(2 * (p - 2))])
    assert np.abs(lf.dtn @ trace - expected).max() <= 1e-11
    assert np.allclose(lf.solve_interior(np.ones(lf.s.shape[0])), lf.solve_interior(np.ones((lf.s.shape[0], 2)))[:, 0])


def test_leaf_factors_one_launch():
    """build_leaf_factors: DtN and S from ONE factorization (hps_leaf_factors): S equals
    the solution-operator launch bit for bit, T the DtN launch to rounding, and both
    the oracle within 1e-10."""
    from paper_2503_04033_b200.engine import LeafEngine
    from paper_2503_04033_b200.local_ops import LeafTemplate
    from oracle import hps_oracle as O
    rng = np.random.default_rng(3)
    for d, p in ((3, 8), (3, 12), (2, 9)):
        tpl = LeafTemplate((0.25,) * d, p, "drop", False)
        n = tpl.n_interior
        pack = np.concatenate([1.0 + 0.05 * rng.standard_normal((3, d, n)),
                               -200.0 * (1.0 + 0.1 * rng.standard_normal((3, 1, n)))], axis=1)
        eng = LeafEngine(tpl, False, True, device=0)
        t, s, stats = eng.factors_host(pack)
        s_ref, _ = eng.solution_operator_host(pack)
        t_ref, _ = eng.dtn_host(pack)
        assert np.array_equal(s, s_ref)
        assert rel(t, t_ref) <= 1e-12
        otpl = O.OracleTemplate(tpl.widths, p)
        for k in range(3):
            ot, os_, _ = O.leaf_dtn(otpl, pack[k, :d].T, None, pack[k, d])
            assert rel(t[k], ot) <= 1e-10 and rel(s[k], os_) <= 1e-10
        assert np.all(stats[:, 0] > 0)


def test_launches_on_different_streams_are_ordered():
    """A device-buffer launch queued on torch's stream and a host-buffer launch (own
    streams) on the same plan do not overlap on the shared slot workspace."""
    import torch
    from paper_2503_04033_b200.engine import LeafEngine
    from paper_2503_04033_b200.local_ops import LeafTemplate
    rng = np.random.default_rng(8)
    tpl = LeafTemplate((0.25,) * 3, 10, "drop", False)
    n = tpl.n_interior
    L = 600
    pack = np.concatenate([np.ones((L, 3, n)), -300.0 * (1.0 + 0.2 * rng.standard_normal((L, 1, n)))],
                          axis=1)
    eng = LeafEngine(tpl, False, True, device=0)
    ref, _ = eng.dtn_host(pack)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        dev, _ = eng.dtn(torch.from_numpy(pack).cuda(), stream=side)   # still running ...
    host, _ = eng.dtn_host(pack[::-1].copy())                          # ... when this starts
    torch.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy(), ref)
    assert np.array_equal(host, ref[::-1])


def test_bench_emits_contract_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--p", "8", "--boxes", "4",
                          "--steps", "3", "--warmup", "3", "--cpu-seconds", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "e2e",
                "roofline", "cpu_baseline", "clocks", "gpu_launches"):
        assert key in line
    assert line["parity"]["max_rel_fro_err_vs_oracle"] <= 1e-10
