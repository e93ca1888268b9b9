"""Host-side mirror of the reference interface (no GPU needed).

Templates, geometry numbering, coefficient packing, schedule resolution and
the pivot rule are checked against the reference's own golden outputs and the
examples of its test-suite (reference tests/test_local_ops.py,
test_geometry.py, test_condensation.py).
"""

import os

import numpy as np
import pytest

from paper_2503_04033_b200 import condensation as cond
from paper_2503_04033_b200.errors import ConfigError, CrossTermError, LeafSingularError
from paper_2503_04033_b200.geometry import (DomainBox, MeshConfig, build_discretization,
                                            leaf_neighbors, sinusoidal_map)
from paper_2503_04033_b200.local_ops import (DROP_CORNERS, LEGENDRE_FACES, LeafTemplate,
                                             cheb_diff_matrix, cheb_nodes, check_pivots,
                                             face_interp_cheb_to_legendre, isotropic_field,
                                             legendre_nodes, pack_coefficients)
from paper_2503_04033_b200.problems import make_problem

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "leaf_cases.npz"))
PG = np.load(os.path.join(HERE, "golden", "pipeline_cases.npz"))
CASES = sorted({k.split("/")[0] for k in G.files})


@pytest.mark.parametrize("name", CASES)
def test_template_matches_reference(name):
    d, p, _, _, leg, hc = (int(x) for x in G[name + "/meta"])
    tpl = LeafTemplate(G[name + "/widths"], p, LEGENDRE_FACES if leg else DROP_CORNERS, bool(hc))
    assert np.array_equal(np.stack(tpl.diff), G[name + "/D"])
    assert np.array_equal(tpl.interior_idx, G[name + "/interior_idx"])
    assert np.array_equal(tpl.a_bi, G[name + "/a_bi"])
    assert np.array_equal(tpl.a_bb, G[name + "/a_bb"])
    if leg:
        assert np.array_equal(tpl._boundary_injection, G[name + "/Q"])
    else:
        assert np.array_equal(tpl._bcols, G[name + "/bcols"])


def test_cheb_nodes_properties():
    x = cheb_nodes(5, (-1.0, 1.0))
    assert x[0] == -1.0 and x[-1] == 1.0
    assert np.allclose(x + x[::-1], 0.0, atol=0.0)
    assert cheb_nodes(3).tolist() == [-1.0, 0.0, 1.0]
    y = cheb_nodes(5, (0.0, 1.0))
    assert y[1] == pytest.approx((1 - np.sqrt(2) / 2) / 2, abs=1e-15)
    with pytest.raises(ValueError):
        cheb_nodes(1)


@pytest.mark.parametrize("p", [2, 3, 5, 8, 13])
def test_diff_matrix_exact_on_polynomials(p):
    D, x = cheb_diff_matrix(p), cheb_nodes(p)
    assert np.abs(D @ np.ones(p)).max() < 1e-13
    assert np.abs(D @ x - 1.0).max() < 1e-12
    for k in range(2, p):
        assert np.abs(D @ x ** k - k * x ** (k - 1)).max() < 1e-10 * p ** 2


def test_face_interp_round_trip():
    for p in (4, 6, 9):
        fwd, rev = face_interp_cheb_to_legendre(p)
        xg = legendre_nodes(p - 1)
        for k in range(p - 1):
            assert np.abs(fwd @ (rev @ xg ** k) - xg ** k).max() < 1e-12 * max(1.0, np.abs(xg ** k).max())
    fwd, rev = face_interp_cheb_to_legendre(5, face_dim=2)
    assert fwd.shape == (16, 25) and np.allclose(fwd.sum(axis=1), 1.0, atol=1e-13)


def test_cross_terms_need_legendre():
    with pytest.raises(CrossTermError):
        LeafTemplate((1.0, 1.0), 6, DROP_CORNERS, True)
    tpl = LeafTemplate((1.0, 1.0, 1.0), 5, LEGENDRE_FACES, True)
    assert tpl.a_bb.shape == (6 * 16, 6 * 16)


def test_geometry_counts():
    disc = build_discretization(DomainBox((0.0, 0.0), (1.0, 1.0)), MeshConfig((1, 1), 6))
    assert disc.index_interior[0].size == 16 and disc.n_interface == 0 and disc.n_dirichlet == 16
    disc = build_discretization(DomainBox((0.0, 0.0), (1.0, 1.0)), MeshConfig((2, 1), 6))
    assert disc.n_interface == 4
    disc = build_discretization(DomainBox((0.0,) * 3, (1.0,) * 3), MeshConfig((2, 2, 2), 8))
    assert disc.n_interface == 432
    nb = leaf_neighbors(build_discretization(DomainBox((0.0, 0.0), (1.0, 1.0)),
                                             MeshConfig((3, 3), 5)), 4)
    assert all(other is not None for _, other in nb)
    with pytest.raises(ConfigError):
        MeshConfig((2, 2), 3)


@pytest.mark.parametrize("name,prob,d,params,boxes,p", [
    ("poisson2_2x2_p6", "poisson_green", 2, {}, (2, 2), 6),
    ("gravity2_3x2_p7", "gravity_helmholtz", 2, {"kappa": 5.0}, (3, 2), 7),
    ("helm3_2x2x2_p6", "helmholtz_green", 3, {"kappa": 6.0}, (2, 2, 2), 6),
    ("convdiff3_2x1x2_p5", "convdiff_step", 3, {}, (2, 1, 2), 5),
    ("curved2_2x2_p6_leg", "curved_helmholtz", 2, {"kappa": 4.0}, (2, 2), 6),
    ("curved3_2x1x1_p5_leg", "curved_helmholtz", 3, {"kappa": 4.0}, (2, 1, 1), 5),
])
def test_numbering_matches_reference(name, prob, d, params, boxes, p):
    spec = make_problem(prob, d=d, **params)
    mode = LEGENDRE_FACES if name.endswith("_leg") else DROP_CORNERS
    disc = build_discretization(spec.domain, MeshConfig(boxes, p, mode))
    assert np.array_equal(disc.nodes, PG[name + "/nodes"])
    if name + "/exact" in PG.files:
        assert np.array_equal(spec.exact(disc.nodes), PG[name + "/exact"])


def test_sinusoidal_map_identity_and_cross_term():
    base = isotropic_field(3, zeroth=lambda x: np.full(x.shape[0], -4.0))
    same = sinusoidal_map(0.0, 6.0).coefficient_transform(base)
    x = np.random.default_rng(0).uniform(size=(20, 3))
    assert np.allclose(same.second_order(x), np.eye(3)[None])
    curved = sinusoidal_map(0.25, 6.0).coefficient_transform(base)
    assert curved.has_cross_terms
    xc = np.array([[np.pi / 12, 0.3, 0.1]])  # psi'(x1) = 0 there
    assert abs(curved.second_order(xc)[0, 0, 1]) < 1e-15
    with pytest.raises(ConfigError):
        sinusoidal_map(1.0, 6.0)


def test_pack_layout_and_pivot_rule():
    f = isotropic_field(3, zeroth=lambda x: x[:, 0], first=lambda x: 2 * x)
    pts = np.random.default_rng(1).uniform(size=(2 * 5, 3))
    pack = pack_coefficients(f, pts, 2)
    assert pack.shape == (2, 7, 5)
    assert np.array_equal(pack[1, 6], pts[5:, 0])
    assert np.array_equal(pack[0, 3], 2 * pts[:5, 0])
    check_pivots(np.array([[1.0, 10.0]]), [(0, 0)])
    with pytest.raises(LeafSingularError):
        check_pivots(np.array([[1.0, 2.0], [1e-15, 1.0]]), [(0,), (1,)])
    with pytest.raises(LeafSingularError):
        check_pivots(np.array([[0.0, 0.0]]), [(0,)])


def test_schedule_resolution():
    n_i, n_b = 18 ** 3, 6 * 18 ** 2
    assert cond.estimate_workspace(20, 3) == 8 * (n_i * n_i + n_i * n_b + n_b * n_b)
    with pytest.raises(ConfigError):
        cond.BatchSchedule(memory_budget=1024).resolve(8, 3, DROP_CORNERS)
    ws = cond.estimate_workspace(6, 2)
    r = cond.BatchSchedule(memory_budget=3 * ws, batch_size=64, workers=8).resolve(6, 2, DROP_CORNERS)
    assert 1 <= r.batch_size and r.batch_size * r.workspace_bytes <= 3 * ws
    r = cond.BatchSchedule().resolve(8, 3, DROP_CORNERS)
    assert r.batch_size * r.workspace_bytes + r.resident_limit * r.block_bytes <= r.memory_budget


def test_cn_fields_and_parabolic_registry():
    from paper_2503_04033_b200.problems import (TimeStepConfig, cn_step_fields,
                                                interior_sample_points, make_parabolic)
    prob = make_parabolic("convection_diffusion", d=3)
    implicit, explicit = cn_step_fields(prob, dt=0.1)
    pts = interior_sample_points(prob.domain, 10, np.random.default_rng(3))
    assert np.allclose(implicit.second_order(pts), -explicit.second_order(pts), atol=0.0)
    assert np.allclose(implicit.first_order(pts), -explicit.first_order(pts), atol=0.0)
    zi, ze = implicit.zeroth_order(pts), explicit.zeroth_order(pts)
    assert np.allclose(zi - 1.0, -(ze - 1.0), atol=1e-15)
    with pytest.raises(ConfigError):
        TimeStepConfig(dt=0.0, t_end=1.0)
    with pytest.raises(ConfigError):
        TimeStepConfig(dt=1.0, t_end=0.5)
    with pytest.raises(ConfigError):
        make_parabolic("nope")
