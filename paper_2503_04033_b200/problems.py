"""Elliptic problem registry (mirror of steklov.problems' elliptic part).

Free-space Green's function problems for Laplace/Helmholtz, the gravity
Helmholtz source problem, the sinusoidally mapped Helmholtz problem, the
implicit convection-diffusion half-step, and the benchmark family of
BASELINE.json configs 2-3: Helmholtz with a Gaussian-bump wave speed b(x).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np
from scipy.special import y0 as bessel_y0

from .errors import ConfigError
from .geometry import DomainBox, ParameterMap, sinusoidal_map
from .local_ops import CoefficientField, isotropic_field

POISSON_DOMAIN_3D = DomainBox(lo=(-1.1, 1.0, 1.2), hi=(0.1, 2.0, 2.2))
POISSON_DOMAIN_2D = DomainBox(lo=(-1.1, 1.0), hi=(0.1, 2.0))
GRAVITY_DOMAIN_3D = DomainBox(lo=(1.1, -1.0, -1.2), hi=(2.1, 0.0, -0.2))
GRAVITY_DOMAIN_2D = DomainBox(lo=(1.1, -1.0), hi=(2.1, 0.0))
CONVDIFF_DOMAIN_3D = DomainBox(lo=(-0.5, -0.5, -0.5), hi=(0.5, 0.5, 0.5))
CONVDIFF_DOMAIN_2D = DomainBox(lo=(-0.5, -0.5), hi=(0.5, 0.5))
UNIT_CUBE = DomainBox(lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0))
UNIT_SQUARE = DomainBox(lo=(0.0, 0.0), hi=(1.0, 1.0))


@dataclass
class ProblemSpec:
    name: str
    coeffs: CoefficientField
    f: Callable[[np.ndarray], np.ndarray]
    g: Callable[[np.ndarray], np.ndarray]
    domain: DomainBox
    exact: Optional[Callable[[np.ndarray], np.ndarray]] = None
    parameter_map: Optional[ParameterMap] = None

    @property
    def requires_legendre_faces(self) -> bool:
        return self.coeffs.has_cross_terms


def _zero(x):
    return np.zeros(x.shape[0])


def _exclude_origin(domain: DomainBox) -> None:
    if all(lo <= 0.0 <= hi for lo, hi in zip(domain.lo, domain.hi)):
        raise ConfigError("domain must exclude the origin for the free-space Green's function")


def _green(d: int, kappa: float):
    if d == 3:
        return lambda x: np.cos(kappa * np.linalg.norm(x, axis=1)) / (4.0 * np.pi * np.linalg.norm(x, axis=1))
    if kappa == 0.0:
        return lambda x: -np.log(np.linalg.norm(x, axis=1)) / (2.0 * np.pi)
    return lambda x: bessel_y0(kappa * np.linalg.norm(x, axis=1))


def poisson_green(domain: Optional[DomainBox] = None, d: int = 3) -> ProblemSpec:
    domain = domain or (POISSON_DOMAIN_3D if d == 3 else POISSON_DOMAIN_2D)
    _exclude_origin(domain)
    exact = _green(domain.d, 0.0)
    return ProblemSpec(name="poisson_green", coeffs=isotropic_field(domain.d), f=_zero, g=exact,
                       exact=exact, domain=domain)


def helmholtz_green(domain: Optional[DomainBox] = None, kappa: float = 16.0,
                    d: int = 3) -> ProblemSpec:
    domain = domain or (POISSON_DOMAIN_3D if d == 3 else POISSON_DOMAIN_2D)
    _exclude_origin(domain)
    kappa = float(kappa)
    exact = _green(domain.d, kappa)
    coeffs = isotropic_field(domain.d, zeroth=lambda x: np.full(x.shape[0], -kappa * kappa))
    return ProblemSpec(name="helmholtz_green", coeffs=coeffs, f=_zero, g=exact, exact=exact,
                       domain=domain)


def gravity_helmholtz(domain: Optional[DomainBox] = None, kappa: float = 12.0,
                      d: int = 3) -> ProblemSpec:
    """Lap u + kappa^2 (1 - x_last) u = -1, u = 0 on the boundary."""
    domain = domain or (GRAVITY_DOMAIN_3D if d == 3 else GRAVITY_DOMAIN_2D)
    kappa, last = float(kappa), domain.d - 1
    coeffs = isotropic_field(domain.d, zeroth=lambda x: -kappa * kappa * (1.0 - x[:, last]))
    return ProblemSpec(name="gravity_helmholtz", coeffs=coeffs,
                       f=lambda x: np.ones(x.shape[0]), g=_zero, domain=domain)


def bump_b(x: np.ndarray, center=0.5, width: float = 0.15, depth: float = 0.5) -> np.ndarray:
    """b(x) = 1 - depth * exp(-|x - c|^2 / (2 width^2)) in (1 - depth, 1]."""
    r2 = ((x - center) ** 2).sum(axis=1)
    return 1.0 - depth * np.exp(-r2 / (2.0 * width * width))


def bump_helmholtz(domain: Optional[DomainBox] = None, kappa: float = 40.0,
                   d: int = 3) -> ProblemSpec:
    """Variable-coefficient Helmholtz -Lap u - kappa^2 b(x) u = 1, u = 0 (BASELINE configs 2-3).

    b(x) is a Gaussian bump with values in (0.5, 1] so kappa^2 b stays below the
    first Dirichlet eigenvalue of a 1/16-wide leaf for kappa <= 80.
    """
    domain = domain or (UNIT_CUBE if d == 3 else UNIT_SQUARE)
    kappa = float(kappa)
    coeffs = isotropic_field(domain.d, zeroth=lambda x: -kappa * kappa * bump_b(x))
    return ProblemSpec(name="bump_helmholtz", coeffs=coeffs, f=lambda x: np.ones(x.shape[0]),
                       g=_zero, domain=domain)


def curved_helmholtz(kappa: float = 16.0, d: int = 3, amplitude: float = 0.25,
                     frequency: float = 6.0, domain: Optional[DomainBox] = None) -> ProblemSpec:
    """Helmholtz on a sinusoidal domain pulled back to a box (needs legendre faces)."""
    domain = domain or (GRAVITY_DOMAIN_3D if d == 3 else GRAVITY_DOMAIN_2D)
    kappa = float(kappa)
    pmap = sinusoidal_map(amplitude, frequency)
    base = isotropic_field(domain.d, zeroth=lambda x: np.full(x.shape[0], -kappa * kappa))
    physical = _green(domain.d, kappa)
    exact = lambda x: physical(pmap.forward(x))  # noqa: E731
    return ProblemSpec(name="curved_helmholtz", coeffs=pmap.coefficient_transform(base), f=_zero,
                       g=exact, exact=exact, domain=domain, parameter_map=pmap)


def _rotation_velocity(d: int):
    def velocity(x):
        b = np.zeros_like(x)
        s = x[:, 2] if d == 3 else 1.0
        b[:, 0] = -np.cos(x[:, 0]) * np.sin(x[:, 1]) * s
        b[:, 1] = np.sin(x[:, 0]) * np.cos(x[:, 1]) * s
        return b
    return velocity


def gaussian_bump(center: Sequence[float], variance: float = 0.002):
    c = np.asarray(center, dtype=float)
    return lambda x: np.exp(-((x - c[None, :]) ** 2).sum(axis=1) / variance)


def convdiff_step(domain: Optional[DomainBox] = None, d: int = 3, dt: float = 0.05,
                  diffusivity: float = 1e-4) -> ProblemSpec:
    """Implicit Crank-Nicolson half-step (I - dt/2 A) of the contaminant model (Eq. 15-16)."""
    prob = convection_diffusion(d=d, diffusivity=diffusivity)
    implicit, _ = cn_step_fields(prob, dt)
    return ProblemSpec(name="convdiff_step", coeffs=implicit, f=prob.u0, g=_zero,
                       domain=domain or prob.domain)


ELLIPTIC_REGISTRY = {
    "poisson_green": poisson_green,
    "helmholtz_green": helmholtz_green,
    "gravity_helmholtz": gravity_helmholtz,
    "bump_helmholtz": bump_helmholtz,
    "curved_helmholtz": curved_helmholtz,
    "convdiff_step": convdiff_step,
}


def make_problem(name: str, d: int = 3, **params) -> ProblemSpec:
    if name not in ELLIPTIC_REGISTRY:
        raise ConfigError(f"unknown problem {name!r}; known: {sorted(ELLIPTIC_REGISTRY)}")
    return ELLIPTIC_REGISTRY[name](d=d, **params)


def relative_l2_error(u: np.ndarray, exact_values: np.ndarray) -> float:
    u = np.asarray(u, dtype=float)
    exact_values = np.asarray(exact_values, dtype=float)
    denom = float(np.linalg.norm(exact_values))
    if denom == 0.0:
        raise ConfigError("reference solution has zero norm")
    return float(np.linalg.norm(u - exact_values)) / denom


# ---------------------------------------------------------------------------
# Parabolic problems and Crank-Nicolson time stepping (reference problems.py:59-86,
# 189-267, 441-515): the implicit operator (I - dt/2 A) is built and factorized
# once; every step applies (I + dt/2 A) to u^n leaf by leaf on the GPU
# (hps_leaf_apply) and runs the solve stage with that load.
# ---------------------------------------------------------------------------

@dataclass
class TimeStepConfig:
    dt: float
    t_end: float
    u0: Optional[Callable[[np.ndarray], np.ndarray]] = None

    def __post_init__(self):
        if not self.dt > 0.0:
            raise ConfigError("dt must be positive")
        if self.t_end < self.dt:
            raise ConfigError("t_end must cover at least one step")

    @property
    def steps(self) -> int:
        return int(round(self.t_end / self.dt))


@dataclass
class ParabolicProblem:
    """du/dt = diffusivity Lap(u) - div(velocity u), homogeneous Dirichlet."""

    name: str
    domain: DomainBox
    diffusivity: float
    velocity: Optional[Callable[[np.ndarray], np.ndarray]] = None
    div_velocity: Optional[Callable[[np.ndarray], np.ndarray]] = None
    u0: Optional[Callable[[np.ndarray], np.ndarray]] = None
    exact: Optional[Callable[[np.ndarray, float], np.ndarray]] = None


def convection_diffusion(d: int = 3, diffusivity: float = 1e-4) -> ParabolicProblem:
    domain = CONVDIFF_DOMAIN_3D if d == 3 else CONVDIFF_DOMAIN_2D
    return ParabolicProblem(name="convection_diffusion", domain=domain,
                            diffusivity=float(diffusivity), velocity=_rotation_velocity(domain.d),
                            div_velocity=_zero, u0=gaussian_bump((0.0, -0.3, 0.0)[:domain.d]))


def heat_manufactured(d: int = 3) -> ParabolicProblem:
    domain = UNIT_CUBE if d == 3 else UNIT_SQUARE
    rate = domain.d * np.pi ** 2

    def exact(x, t):
        return math.exp(-rate * t) * np.prod(np.sin(np.pi * x), axis=1)

    return ParabolicProblem(name="heat_manufactured", domain=domain, diffusivity=1.0,
                            u0=lambda x: exact(x, 0.0), exact=exact)


def cn_step_fields(prob: ParabolicProblem, dt: float):
    """(implicit, explicit) coefficient fields of (I -+ dt/2 A), Eq. (16)."""
    def make(sign: float) -> CoefficientField:
        half = sign * 0.5 * dt
        first = None
        if prob.velocity is not None:
            vel = prob.velocity
            first = lambda x, _h=half: _h * vel(x)  # noqa: E731
        div_v = prob.div_velocity

        def zeroth(x, _h=half):
            out = np.ones(x.shape[0])
            return out + _h * div_v(x) if div_v is not None else out

        return isotropic_field(prob.domain.d, diffusion=half * prob.diffusivity, zeroth=zeroth,
                               first=first)
    return make(1.0), make(-1.0)


PARABOLIC_REGISTRY = {"heat_manufactured": heat_manufactured,
                      "convection_diffusion": convection_diffusion}


def make_parabolic(name: str, d: int = 3, **params) -> ParabolicProblem:
    if name not in PARABOLIC_REGISTRY:
        raise ConfigError(f"unknown parabolic problem {name!r}; known: {sorted(PARABOLIC_REGISTRY)}")
    return PARABOLIC_REGISTRY[name](d=d, **params)


@dataclass
class Trajectory:
    times: list
    states: list
    factorization_events: int
    step_seconds: list
    system: object

    @property
    def final(self) -> np.ndarray:
        return self.states[-1]


def crank_nicolson_run(disc, prob: ParabolicProblem, cfg: TimeStepConfig, schedule=None,
                       snapshot_stride: int = 1) -> Trajectory:
    """Advance a parabolic problem; the implicit operator is factorized once."""
    import time as _time
    from . import condensation
    from .condensation import BatchSchedule, interior_points
    from .engine import LeafEngine
    from .local_ops import DROP_CORNERS, pack_coefficients

    if snapshot_stride < 1:
        raise ConfigError("snapshot stride must be >= 1")
    if disc.corner_mode != DROP_CORNERS:
        raise ConfigError("time stepping uses corner-dropping meshes "
                          "(the step operators have no cross terms)")
    implicit, explicit = cn_step_fields(prob, cfg.dt)
    sys = condensation.build(disc, implicit, schedule or BatchSchedule(cache_leaf_factors=True))
    engine = LeafEngine.for_template(sys.template, explicit, device=sys.schedule.device)
    leaves = range(len(disc.leaves))
    pack_ex = pack_coefficients(explicit, interior_points(disc, leaves), len(disc.leaves))
    int_ids = np.stack([lf.interior_ids for lf in disc.leaves])
    bnd_ids = np.stack([lf.boundary_ids for lf in disc.leaves])
    u0 = cfg.u0 or prob.u0
    if u0 is None:
        raise ConfigError("no initial condition available")
    u = np.asarray(u0(disc.nodes), dtype=float).copy()
    times, states, step_seconds = [0.0], [u.copy()], []
    for step in range(1, cfg.steps + 1):
        tic = _time.perf_counter()
        w = np.zeros(disc.n_total)
        w[int_ids] = engine.apply_host(pack_ex, u[int_ids], u[bnd_ids])
        u = condensation.run_solve_stage(sys, w, _zero).u
        step_seconds.append(_time.perf_counter() - tic)
        if step % snapshot_stride == 0 or step == cfg.steps:
            times.append(step * cfg.dt)
            states.append(u.copy())
    return Trajectory(times=times, states=states, factorization_events=1,
                      step_seconds=step_seconds, system=sys)


def interior_sample_points(domain: DomainBox, n: int, rng=None, margin: float = 0.05) -> np.ndarray:
    """Random points strictly inside the domain (reference problems.py:371-378)."""
    rng = rng or np.random.default_rng(0)
    lo, hi = np.asarray(domain.lo), np.asarray(domain.hi)
    pad = margin * (hi - lo)
    return rng.uniform(lo + pad, hi - pad, size=(n, domain.d))


def plane_mass_center(u: np.ndarray, nodes: np.ndarray, split_axis: int = 2) -> np.ndarray:
    """Density-weighted (x1, x2) center of the upper half (x_split > 0), weights clipped at 0."""
    mask = nodes[:, split_axis] > 0.0 if nodes.shape[1] > split_axis else slice(None)
    w = np.clip(u[mask], 0.0, None)
    total = w.sum()
    if total <= 0.0:
        raise ConfigError("no positive mass in the upper half domain")
    return (w[:, None] * nodes[mask][:, :2]).sum(axis=0) / total


def unwrap_angles(centers) -> np.ndarray:
    return np.unwrap(np.array([math.atan2(c[1], c[0]) for c in centers]))
