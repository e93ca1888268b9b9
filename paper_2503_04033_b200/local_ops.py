"""Per-leaf operators: host templates and the GPU-backed leaf factors.

Mirrors ``steklov.local_ops`` (reference: local_ops.py).  The small,
operator-independent pieces (Chebyshev nodes, differentiation matrices, the
index partition of a leaf grid, the shared normal-derivative blocks a_bi /
a_bb) are built once on the host in float64 — they are O(p^2 .. p^(2d-1)) and
shared by every leaf.  Everything per leaf (operator assembly, pivoted LU of
A_ii, DtN map, solution operator, interior solves) runs in the CUDA engine
(:mod:`paper_2503_04033_b200.engine`); there is no CPU implementation of those.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np

from .errors import CrossTermError, LeafSingularError

DROP_CORNERS = "drop"
LEGENDRE_FACES = "legendre"
CORNER_MODES = (DROP_CORNERS, LEGENDRE_FACES)

PIVOT_FLOOR = 1e-14  # relative pivot floor of factor_interior (local_ops.py:32)


# ---------------------------------------------------------------------------
# 1D spectral primitives (reference local_ops.py:39-136)
# ---------------------------------------------------------------------------

def _lobatto_weights(p: int) -> np.ndarray:
    w = np.where(np.arange(p) % 2 == 0, 1.0, -1.0)
    w[[0, -1]] *= 0.5
    return w


def cheb_nodes(p: int, interval: Sequence[float] = (-1.0, 1.0)) -> np.ndarray:
    """Chebyshev–Lobatto points ascending on [a, b], endpoints exact.

    sin(pi (2j - n) / (2n)) is antisymmetric in floating point, so the grid is
    symmetric about the midpoint (reference local_ops.py:39-55).
    """
    if p < 2:
        raise ValueError(f"need at least 2 nodes per dimension, got p={p}")
    lo, hi = float(interval[0]), float(interval[1])
    n = p - 1
    s = np.sin(np.pi * (2 * np.arange(p) - n) / (2 * n))
    x = 0.5 * (lo + hi) + 0.5 * (hi - lo) * s
    x[0], x[-1] = lo, hi
    return x


def cheb_diff_matrix(p: int) -> np.ndarray:
    """Differentiation matrix on the p-point Lobatto grid of [-1, 1].

    Off-diagonal barycentric formula, diagonal = minus the row sum
    (reference local_ops.py:58-73).
    """
    if p < 2:
        raise ValueError(f"need at least 2 nodes, got p={p}")
    x = cheb_nodes(p)
    w = _lobatto_weights(p)
    gap = x[:, None] - x[None, :]
    np.fill_diagonal(gap, 1.0)
    D = (w[None, :] / w[:, None]) / gap
    np.fill_diagonal(D, 0.0)
    np.fill_diagonal(D, -D.sum(axis=1))
    return D


def legendre_nodes(n: int, interval: Sequence[float] = (-1.0, 1.0)) -> np.ndarray:
    """Gauss–Legendre points on [a, b] (reference local_ops.py:76-82)."""
    if n < 1:
        raise ValueError(f"need at least 1 node, got n={n}")
    lo, hi = float(interval[0]), float(interval[1])
    t, _ = np.polynomial.legendre.leggauss(n)
    return 0.5 * (lo + hi) + 0.5 * (hi - lo) * t


def interp_matrix(src: np.ndarray, dst: np.ndarray,
                  weights: Optional[np.ndarray] = None) -> np.ndarray:
    """Barycentric Lagrange interpolation from nodes ``src`` to points ``dst``."""
    src = np.asarray(src, dtype=float)
    dst = np.asarray(dst, dtype=float)
    if weights is None:
        gap = src[:, None] - src[None, :]
        np.fill_diagonal(gap, 1.0)
        weights = 1.0 / gap.prod(axis=1)
        weights = weights / np.abs(weights).max()
    out = np.zeros((dst.size, src.size))
    for i, t in enumerate(dst):
        exact = np.flatnonzero(src == t)
        if exact.size:
            out[i, exact[0]] = 1.0
        else:
            c = weights / (t - src)
            out[i] = c / c.sum()
    return out


def face_interp_cheb_to_legendre(p: int, face_dim: int = 1):
    """(forward, reverse) tensor interpolation between Chebyshev and Gauss face grids."""
    if p < 4:
        raise ValueError(f"face reinterpolation needs p >= 4, got p={p}")
    fwd1 = interp_matrix(cheb_nodes(p), legendre_nodes(p - 1), weights=_lobatto_weights(p))
    rev1 = interp_matrix(legendre_nodes(p - 1), cheb_nodes(p))
    fwd, rev = fwd1, rev1
    for _ in range(face_dim - 1):
        fwd, rev = np.kron(fwd, fwd1), np.kron(rev, rev1)
    return fwd, rev


# ---------------------------------------------------------------------------
# Coefficient fields (reference local_ops.py:143-190)
# ---------------------------------------------------------------------------

@dataclass
class CoefficientField:
    """Coefficients of  -sum a_ij d2u/dxi dxj + sum b_i du/dxi + c u.

    Callables take (n, d) points and return (n, d, d), (n, d) and (n,) arrays.
    """

    second_order: Callable[[np.ndarray], np.ndarray]
    first_order: Optional[Callable[[np.ndarray], np.ndarray]] = None
    zeroth_order: Optional[Callable[[np.ndarray], np.ndarray]] = None
    has_cross_terms: bool = False

    def validate_cross_flag(self, points: np.ndarray) -> None:
        a2 = np.asarray(self.second_order(points))
        off = a2 * (1.0 - np.eye(points.shape[1]))[None]
        if np.any(off != 0.0) and not self.has_cross_terms:
            raise CrossTermError(
                "second_order has off-diagonal entries but has_cross_terms is False")


def isotropic_field(d: int, diffusion: float = 1.0, zeroth=None, first=None) -> CoefficientField:
    """diffusion * (-Laplace) plus optional first/zeroth order terms."""
    eye = diffusion * np.eye(d)
    return CoefficientField(second_order=lambda x: np.broadcast_to(eye, (x.shape[0], d, d)),
                            first_order=first, zeroth_order=zeroth)


def laplace_field(d: int) -> CoefficientField:
    return isotropic_field(d)


# ---------------------------------------------------------------------------
# Leaf template (reference local_ops.py:206-353)
# ---------------------------------------------------------------------------

class LeafTemplate:
    """Operator-independent data shared by all equal leaves of one mesh.

    Grid multi-indices are C ordered (axis 0 slowest).  Faces are ordered
    -x, +x, -y, +y[, -z, +z]; nodes inside a face lexicographically.
    ``drop`` keeps face-interior Chebyshev nodes as boundary DOFs;
    ``legendre`` keeps (p-1)^(d-1) Gauss nodes per face.
    """

    def __init__(self, widths: Sequence[float], p: int, corner_mode: str, cross_terms: bool):
        if corner_mode not in CORNER_MODES:
            raise ValueError(f"unknown corner mode {corner_mode!r}")
        if cross_terms and corner_mode == DROP_CORNERS:
            raise CrossTermError("cross-derivative terms require Legendre face grids; "
                                 "corner nodes cannot simply be dropped")
        self.widths = tuple(float(w) for w in widths)
        self.d = d = len(self.widths)
        self.p = p = int(p)
        self.corner_mode = corner_mode
        self.cross_terms = bool(cross_terms)
        self.n_grid = p ** d
        self.ref_offsets = 0.5 * (cheb_nodes(p) + 1.0)
        self.ref_offsets[0], self.ref_offsets[-1] = 0.0, 1.0
        self.diff = [cheb_diff_matrix(p) * (2.0 / w) for w in self.widths]
        self.diff2 = [D @ D for D in self.diff]

        multi = np.indices((p,) * d).reshape(d, -1)
        at_end = (multi == 0) | (multi == p - 1)
        self.end_count = at_end.sum(axis=0)
        self.interior_idx = np.flatnonzero(self.end_count == 0)
        self.n_interior = self.interior_idx.size
        self.boundary_all_idx = np.flatnonzero(self.end_count > 0)
        self.face_node_idx, self.face_full_idx, self.face_axes = [], [], []
        for axis in range(d):
            tangential_inner = ~np.any(np.delete(at_end, axis, axis=0), axis=0)
            for side in (0, 1):
                plane = multi[axis] == side * (p - 1)
                self.face_node_idx.append(np.flatnonzero(plane & tangential_inner))
                self.face_full_idx.append(np.flatnonzero(plane))
                self.face_axes.append((axis, side))
        self.face_dofs = (p - 2) ** (d - 1) if corner_mode == DROP_CORNERS else (p - 1) ** (d - 1)
        self.n_boundary = 2 * d * self.face_dofs
        self.face_slices = [slice(k * self.face_dofs, (k + 1) * self.face_dofs)
                            for k in range(2 * d)]
        self._multi = multi
        if corner_mode == DROP_CORNERS:
            self._bcols = np.concatenate(self.face_node_idx)
            normal = self._normal_rows_drop()
            self.a_bi = np.ascontiguousarray(normal[:, self.interior_idx])
            self.a_bb = np.ascontiguousarray(normal[:, self._bcols])
            self.gauss_offsets = None
        else:
            xc, xg = cheb_nodes(p), legendre_nodes(p - 1)
            self._fwd1 = interp_matrix(xc, xg, weights=_lobatto_weights(p))
            self._rev1 = interp_matrix(xg, xc)
            self.gauss_offsets = 0.5 * (xg + 1.0)
            self._bcols = None
            normal = self._normal_rows_legendre()
            self._boundary_injection = self._injection()
            self.a_bi = np.ascontiguousarray(normal[:, self.interior_idx])
            self.a_bb = normal[:, self.boundary_all_idx] @ self._boundary_injection

    def _normal_rows_drop(self) -> np.ndarray:
        """Signed normal-derivative rows at face-interior nodes over the full grid."""
        p, d, multi = self.p, self.d, self._multi
        rows = []
        for k, (axis, side) in enumerate(self.face_axes):
            sign = 1.0 if side == 1 else -1.0
            edge = p - 1 if side == 1 else 0
            nodes = self.face_node_idx[k]
            block = np.zeros((nodes.size, self.n_grid))
            tang = np.delete(multi, axis, axis=0)
            for r, node in enumerate(nodes):
                on_line = np.all(tang == tang[:, node:node + 1], axis=0)
                cols = np.flatnonzero(on_line)
                block[r, cols] = sign * self.diff[axis][edge, multi[axis, cols]]
            rows.append(block)
        return np.vstack(rows)

    def _normal_rows_legendre(self) -> np.ndarray:
        p, d = self.p, self.d
        blocks = []
        for axis, side in self.face_axes:
            sign = 1.0 if side == 1 else -1.0
            edge = p - 1 if side == 1 else 0
            mat = None
            for dim in range(d):
                part = sign * self.diff[axis][edge:edge + 1, :] if dim == axis else self._fwd1
                mat = part if mat is None else np.kron(mat, part)
            blocks.append(mat)
        return np.vstack(blocks)

    def _injection(self) -> np.ndarray:
        """Gauss face data -> all Chebyshev boundary nodes, edge/corner averaged."""
        pos = np.full(self.n_grid, -1)
        pos[self.boundary_all_idx] = np.arange(self.boundary_all_idx.size)
        rev = self._rev1
        for _ in range(self.d - 2):
            rev = np.kron(rev, self._rev1)
        Q = np.zeros((self.boundary_all_idx.size, self.n_boundary))
        for k in range(2 * self.d):
            full = self.face_full_idx[k]
            Q[pos[full], self.face_slices[k]] += (1.0 / self.end_count[full])[:, None] * rev
        return Q

    def leaf_grid(self, nodes1d: Sequence[np.ndarray]) -> np.ndarray:
        """(p^d, d) coordinates of a leaf's tensor grid, C ordered."""
        mesh = np.meshgrid(*nodes1d, indexing="ij")
        return np.stack([g.reshape(-1) for g in mesh], axis=1)

    def leaf_nodes1d(self, lo: Sequence[float], hi: Sequence[float]):
        out = []
        for k in range(self.d):
            x = lo[k] + (hi[k] - lo[k]) * self.ref_offsets
            x[0], x[-1] = lo[k], hi[k]
            out.append(x)
        return out


# ---------------------------------------------------------------------------
# Coefficient packing for the device (layout of include/hps_leaf.h)
# ---------------------------------------------------------------------------

def coefficient_layout(coeffs: CoefficientField):
    """(has_first, has_zeroth, has_cross) of a field's device coefficient pack."""
    return (coeffs.first_order is not None, coeffs.zeroth_order is not None,
            bool(coeffs.has_cross_terms))


def pack_coefficients(coeffs: CoefficientField, x_int: np.ndarray, n_leaves: int,
                      out: Optional[np.ndarray] = None) -> np.ndarray:
    """Evaluate the coefficient callables at interior nodes of ``n_leaves`` leaves.

    x_int: (n_leaves * n, d) points, leaf-major.  Returns (n_leaves, ncoef, n)
    with rows [a_00 .. a_dd (diagonal second order), a_ab + a_ba for the pairs
    (0,1), (0,2), (1,2) if the field has cross terms (the sum the reference
    forms in collocation_rows, local_ops.py:375-378), b_0 .. b_d, c].
    """
    d = x_int.shape[1]
    n = x_int.shape[0] // max(n_leaves, 1)
    has_first, has_zeroth, has_cross = coefficient_layout(coeffs)
    npair = d * (d - 1) // 2 if has_cross else 0
    ncoef = d + npair + (d if has_first else 0) + (1 if has_zeroth else 0)
    if out is None:
        out = np.empty((n_leaves, ncoef, n))
    a2 = np.asarray(coeffs.second_order(x_int), dtype=float)
    for k in range(d):
        out[:, k, :] = a2[:, k, k].reshape(n_leaves, n)
    row = d
    if has_cross:
        for a in range(d):
            for b in range(a + 1, d):
                out[:, row, :] = (a2[:, a, b] + a2[:, b, a]).reshape(n_leaves, n)
                row += 1
    if has_first:
        a1 = np.asarray(coeffs.first_order(x_int), dtype=float)
        for k in range(d):
            out[:, row + k, :] = a1[:, k].reshape(n_leaves, n)
        row += d
    if has_zeroth:
        out[:, row, :] = np.asarray(coeffs.zeroth_order(x_int), dtype=float).reshape(n_leaves, n)
    return out


def check_pivots(stats: np.ndarray, leaf_indices) -> None:
    """Reference singularity rule of factor_interior (local_ops.py:430-435)."""
    stats = np.asarray(stats)
    dmin, dmax = stats[:, 0], stats[:, 1]
    bad = (dmax == 0.0) | ~np.isfinite(dmin) | ~np.isfinite(dmax) | (dmin <= PIVOT_FLOOR * dmax)
    if np.any(bad):
        k = int(np.flatnonzero(bad)[0])
        if dmax[k] == 0.0:
            detail = "interior block is zero"
        else:
            detail = f"pivot ratio {dmin[k] / dmax[k]:.2e}"
        raise LeafSingularError(leaf_indices[k], detail)


# ---------------------------------------------------------------------------
# Leaf factors (reference local_ops.py:401-463), computed on the GPU
# ---------------------------------------------------------------------------

@dataclass
class LeafFactors:
    """DtN map and solution operator of one leaf, produced by the CUDA engine.

    ``a_ii_factor`` is not materialised: the engine re-factors A_ii on the
    device whenever an interior solve is requested (the paper's recompute
    strategy, §3.2).  ``solve_interior`` therefore needs the coefficient pack.
    """

    a_ii_factor: object
    a_ib: Optional[np.ndarray]
    a_bi: np.ndarray
    a_bb: np.ndarray
    s: np.ndarray
    dtn: np.ndarray
    _engine: object = None
    _coeffs: Optional[np.ndarray] = None

    def solve_interior(self, rhs: np.ndarray) -> np.ndarray:
        rhs = np.asarray(rhs, dtype=float)
        if rhs.ndim == 1:
            return self._engine.reduce_load_host(self._coeffs[None], rhs[None])[0][0]
        k = rhs.shape[1]
        packs = np.repeat(self._coeffs[None], k, axis=0)
        return self._engine.reduce_load_host(packs, np.ascontiguousarray(rhs.T))[0].T


def build_leaf_factors(template: LeafTemplate, coeffs: CoefficientField,
                       grid: np.ndarray, leaf_index=None, engine=None) -> LeafFactors:
    """GPU leaf build: DtN and S for one leaf (reference local_ops.py:439-446)."""
    from .engine import LeafEngine
    x_int = grid[template.interior_idx]
    engine = engine or LeafEngine.for_template(template, coeffs)
    pack = pack_coefficients(coeffs, x_int, 1)
    dtn, s, stats = engine.factors_host(pack)   # one factorization, one launch
    check_pivots(stats, [leaf_index])
    return LeafFactors(a_ii_factor=None, a_ib=None, a_bi=template.a_bi, a_bb=template.a_bb,
                       s=s[0], dtn=dtn[0], _engine=engine, _coeffs=pack[0])


def build_leaf_operator(bounds, p: int, coeffs: CoefficientField,
                        corner_mode: str = DROP_CORNERS) -> LeafFactors:
    """Standalone leaf build from physical bounds (lo, hi) (local_ops.py:449-463)."""
    lo = np.asarray(bounds[0], dtype=float)
    hi = np.asarray(bounds[1], dtype=float)
    template = LeafTemplate(hi - lo, p, corner_mode, coeffs.has_cross_terms)
    grid = template.leaf_grid(template.leaf_nodes1d(lo, hi))
    coeffs.validate_cross_flag(grid[template.interior_idx])
    return build_leaf_factors(template, coeffs, grid, leaf_index=None)
