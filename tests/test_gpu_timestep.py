"""Crank-Nicolson driver on the GPU path (reference acceptance criterion 7)."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_zero_operator_keeps_state():
    """A = 0: both half-step operators are the identity; the polynomial state
    vanishes on the boundary and is represented exactly (reference test_problems.py:148-160)."""
    from paper_2503_04033_b200 import (MeshConfig, TimeStepConfig, build_discretization,
                                       crank_nicolson_run, make_parabolic)
    prob = make_parabolic("heat_manufactured", d=2)
    prob.diffusivity = 0.0
    poly = lambda x: (x[:, 0] * (1 - x[:, 0])) * (x[:, 1] * (1 - x[:, 1]))  # noqa: E731
    disc = build_discretization(prob.domain, MeshConfig((2, 2), 6))
    traj = crank_nicolson_run(disc, prob, TimeStepConfig(dt=0.1, t_end=0.3, u0=poly))
    assert traj.factorization_events == 1 and len(traj.step_seconds) == 3
    scale = np.abs(traj.states[0]).max()
    for state in traj.states[1:]:
        assert np.abs(state - traj.states[0]).max() <= 1e-11 * scale


def test_contaminant_rotates_counterclockwise():
    """Eq. (15) transport model: the mass center turns counterclockwise (Fig. 10)."""
    from paper_2503_04033_b200 import (MeshConfig, TimeStepConfig, build_discretization,
                                       crank_nicolson_run, make_parabolic)
    from paper_2503_04033_b200.problems import plane_mass_center, unwrap_angles
    prob = make_parabolic("convection_diffusion", d=3)
    disc = build_discretization(prob.domain, MeshConfig((3, 3, 3), 10))
    traj = crank_nicolson_run(disc, prob, TimeStepConfig(dt=0.1, t_end=2.5, u0=prob.u0),
                              snapshot_stride=5)
    angles = unwrap_angles([plane_mass_center(s, disc.nodes) for s in traj.states])
    assert (np.diff(angles) > 0.0).all()


def test_heat_temporal_order_two():
    from paper_2503_04033_b200 import (MeshConfig, TimeStepConfig, build_discretization,
                                       crank_nicolson_run, make_parabolic)
    prob = make_parabolic("heat_manufactured", d=2)
    disc = build_discretization(prob.domain, MeshConfig((2, 2), 12))
    t_end = 0.1
    errs = []
    for dt in (0.05, 0.025, 0.0125):
        traj = crank_nicolson_run(disc, prob, TimeStepConfig(dt=dt, t_end=t_end))
        exact = prob.exact(disc.nodes, t_end)
        errs.append(np.linalg.norm(traj.final - exact) / np.linalg.norm(exact))
        assert traj.factorization_events == 1
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert all(1.7 <= o <= 2.3 for o in orders), (errs, orders)
