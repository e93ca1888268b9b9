"""CPU oracle for the HPS leaf-box reduction — TEST INFRASTRUCTURE ONLY.

This module is the *checker* for the CUDA leaf path of ``paper_2503_04033_b200``.
Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import it.  The product package
never imports it and has no CPU fallback.

It restates, in plain numpy/scipy, the algorithm of the reference package
``steklov`` (``/root/reference/pkg/src/steklov``) for the per-leaf path:

* 1D Chebyshev primitives        — local_ops.py:39-73  (cheb_nodes, cheb_diff_matrix,
                                   _lobatto_bary_weights 85-90)
* leaf index partition / faces   — local_ops.py:238-271 (LeafTemplate.__init__)
* normal-derivative blocks       — local_ops.py:302-315 (a_bi, a_bb in ``drop`` mode)
* interior collocation rows      — local_ops.py:362-398 (collocation_rows, interior_blocks)
* pivoted LU + singular guard    — local_ops.py:422-436 (factor_interior, _PIVOT_FLOOR=1e-14)
* DtN / solution operator        — local_ops.py:439-446 (build_leaf_factors)
* load reduction leaf task       — condensation.py:314-323 (reduce_load.leaf_task)
* interior reconstruction task   — condensation.py:372-383 (solve.leaf_task, recompute branch)

The restatement assembles the dense blocks directly from tensor indices (no
scipy.sparse Kronecker chains), but keeps the reference's summation order
(second-order x, y, z; cross; first-order x, y, z; zeroth) so entries agree
bit-for-bit with the reference on the same machine.  Parity is PINNED against
golden vectors produced by the reference itself (``tests/golden/make_golden.py``,
fixtures ``tests/golden/*.npz``; check: ``tests/test_oracle_golden.py``).
"""

from __future__ import annotations

import math
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.linalg

PIVOT_FLOOR = 1e-14  # local_ops.py:32


# --------------------------------------------------------------------------
# 1D spectral primitives (local_ops.py:39-90)
# --------------------------------------------------------------------------

def cheb_points(p, a=-1.0, b=1.0):
    """Chebyshev-Lobatto nodes, ascending, endpoints pinned (local_ops.py:39-55)."""
    k = np.arange(p)
    half = (p - 1)
    t = np.sin(np.pi * (2 * k - half) / (2 * half))
    x = 0.5 * (a + b) + 0.5 * (b - a) * t
    x[0], x[-1] = a, b
    return x


def cheb_D(p):
    """Barycentric differentiation matrix on [-1, 1] (local_ops.py:58-73, 85-90)."""
    x = cheb_points(p)
    w = np.ones(p)
    w[1::2] = -1.0
    w[0] *= 0.5
    w[-1] *= 0.5
    delta = x[:, None] - x[None, :]
    np.fill_diagonal(delta, 1.0)
    D = (w[None, :] / w[:, None]) / delta
    np.fill_diagonal(D, 0.0)
    np.fill_diagonal(D, -D.sum(axis=1))
    return D


# --------------------------------------------------------------------------
# Leaf template (drop-corner mode): index partition + normal blocks
# --------------------------------------------------------------------------

def _bary(x):
    gap = x[:, None] - x[None, :]
    np.fill_diagonal(gap, 1.0)
    w = 1.0 / gap.prod(axis=1)
    return w / np.abs(w).max()


def _interp(src, dst, w):
    """Barycentric interpolation matrix (local_ops.py:100-114)."""
    M = np.zeros((dst.size, src.size))
    for i, t in enumerate(dst):
        hit = np.flatnonzero(src == t)
        if hit.size:
            M[i, hit[0]] = 1.0
        else:
            c = w / (t - src)
            M[i] = c / c.sum()
    return M


class OracleTemplate:
    """Index bookkeeping of one leaf (local_ops.py:238-306).

    Multi-indices are full-grid (0..p-1 per axis, C order, axis 0 slowest).
    ``mode`` "drop": face-interior Chebyshev boundary DOFs; "legendre":
    (p-1)^(d-1) Gauss nodes per face, boundary data injected by the
    averaged tensor interpolation Q (local_ops.py:289-353).
    """

    def __init__(self, widths, p, mode="drop"):
        self.mode = mode
        if mode == "legendre":
            self._init_legendre(widths, p)
            return
        self.widths = tuple(float(w) for w in widths)
        self.d = d = len(self.widths)
        self.p = p
        self.D1 = [cheb_D(p) * (2.0 / w) for w in self.widths]
        self.D2 = [D @ D for D in self.D1]
        grid = np.indices((p,) * d).reshape(d, -1).T          # (p^d, d)
        on_end = (grid == 0) | (grid == p - 1)
        n_end = on_end.sum(axis=1)
        self.interior = grid[n_end == 0]                        # (n, d)
        faces = []
        for axis in range(d):
            tangential_ok = np.all(~np.delete(on_end, axis, axis=1), axis=1)
            for side in (0, 1):
                sel = (grid[:, axis] == side * (p - 1)) & tangential_ok
                faces.append((axis, side, grid[sel]))
        self.faces = faces
        self.boundary = np.concatenate([f[2] for f in faces])   # (m, d)
        self.n = self.interior.shape[0]
        self.m = self.boundary.shape[0]
        self.face_dofs = (p - 2) ** (d - 1)
        # a_bi / a_bb: signed one-sided normal derivative at face nodes
        # (local_ops.py:310-315): row = face node, entry = sign * D1[axis][edge, k]
        # along the normal line through that node.
        self.a_bi = self._normal_block(self.interior)
        self.a_bb = self._normal_block(self.boundary)

    def _init_legendre(self, widths, p):
        self.widths = tuple(float(w) for w in widths)
        self.d = d = len(self.widths)
        self.p = p
        self.D1 = [cheb_D(p) * (2.0 / w) for w in self.widths]
        self.D2 = [D @ D for D in self.D1]
        grid = np.indices((p,) * d).reshape(d, -1).T
        on_end = (grid == 0) | (grid == p - 1)
        n_end = on_end.sum(axis=1)
        self.interior = grid[n_end == 0]
        self.bnd_all = grid[n_end > 0]
        xc = cheb_points(p)
        xg, _ = np.polynomial.legendre.leggauss(p - 1)
        w_lob = np.where(np.arange(p) % 2 == 0, 1.0, -1.0)
        w_lob[[0, -1]] *= 0.5
        fwd1 = _interp(xc, xg, w_lob)
        rev1 = _interp(xg, xc, _bary(xg))
        fd = (p - 1) ** (d - 1)
        self.n, self.m = self.interior.shape[0], 2 * d * fd
        self.face_dofs = fd
        rev_face = rev1 if d == 2 else np.kron(rev1, rev1)
        strides = p ** np.arange(d - 1, -1, -1)
        pos = np.full(p ** d, -1)
        pos[self.bnd_all @ strides] = np.arange(self.bnd_all.shape[0])
        Q = np.zeros((self.bnd_all.shape[0], self.m))
        normal = []
        k = 0
        for axis in range(d):
            for side in (0, 1):
                plane = grid[grid[:, axis] == side * (p - 1)]
                Q[pos[plane @ strides], k * fd:(k + 1) * fd] += \
                    (1.0 / n_end[plane @ strides])[:, None] * rev_face
                sign = 1.0 if side else -1.0
                edge = p - 1 if side else 0
                mat = None
                for dim in range(d):
                    part = sign * self.D1[axis][edge:edge + 1, :] if dim == axis else fwd1
                    mat = part if mat is None else np.kron(mat, part)
                normal.append(mat)
                k += 1
        self.Q = Q
        normal = np.vstack(normal)
        self.a_bi = normal[:, self.interior @ strides]
        self.a_bb = normal[:, self.bnd_all @ strides] @ Q

    def _normal_block(self, cols):
        rows = []
        for axis, side, nodes in self.faces:
            sign = 1.0 if side == 1 else -1.0
            edge = (self.p - 1) if side == 1 else 0
            same_line = np.all(
                np.delete(nodes, axis, axis=1)[:, None, :]
                == np.delete(cols, axis, axis=1)[None, :, :], axis=2)
            vals = sign * self.D1[axis][edge, cols[:, axis]]
            rows.append(np.where(same_line, vals[None, :], 0.0))
        return np.vstack(rows)


def coefficient_count(d, has_first, has_zeroth):
    return d + (d if has_first else 0) + (1 if has_zeroth else 0)


def interior_blocks(tpl, a2diag, a1=None, a0=None, cross=None):
    """Dense (A_ii, A_ib) from coefficients at interior nodes (local_ops.py:362-398).

    a2diag: (n, d) diagonal second-order coefficients; cross: (n, npairs)
    sums a_ab + a_ba for pairs (0,1), (0,2), (1,2) or None; a1: (n, d) or
    None; a0: (n,) or None.  Summation order follows collocation_rows().
    """
    if tpl.mode == "legendre":
        return _interior_blocks_legendre(tpl, a2diag, a1, a0, cross)
    p, d = tpl.p, tpl.d
    R = tpl.interior
    n = R.shape[0]
    strides = p ** np.arange(d - 1, -1, -1)
    # full-grid flat id -> column position in A_ii / A_ib (or -1)
    pos_i = np.full(p ** d, -1)
    pos_i[tpl.interior @ strides] = np.arange(n)
    pos_b = np.full(p ** d, -1)
    pos_b[tpl.boundary @ strides] = np.arange(tpl.m)
    a_ii = np.zeros((n, n))
    a_ib = np.zeros((n, tpl.m))
    rows = np.repeat(np.arange(n), p)
    along = np.tile(np.arange(p), n)

    def scatter(axis, coef, D):
        nbr = np.repeat(R, p, axis=0)
        nbr[:, axis] = along
        flat = nbr @ strides
        vals = coef[rows] * D[R[rows, axis], along]
        for A, pos in ((a_ii, pos_i), (a_ib, pos_b)):
            hit = pos[flat] >= 0
            A[rows[hit], pos[flat[hit]]] += vals[hit]

    for axis in range(d):
        scatter(axis, -a2diag[:, axis], tpl.D2[axis])
    if a1 is not None:
        for axis in range(d):
            scatter(axis, a1[:, axis], tpl.D1[axis])
    if a0 is not None:
        a_ii[np.arange(n), np.arange(n)] += a0
    return a_ii, a_ib


def _interior_blocks_legendre(tpl, a2diag, a1, a0, cross):
    """Full collocation rows over the p^d grid, then A_ii and A_ib = R_b Q."""
    p, d = tpl.p, tpl.d
    R = tpl.interior
    n = R.shape[0]
    strides = p ** np.arange(d - 1, -1, -1)
    full = np.zeros((n, p ** d))
    rows = np.arange(n)

    def add(coef, axes, mats):
        # nodes that differ from the row node only in `axes`
        grids = np.meshgrid(*[np.arange(p)] * len(axes), indexing="ij")
        combos = np.stack([g.reshape(-1) for g in grids], axis=1)
        for combo in combos:
            J = R.copy()
            val = np.ones(n)
            for ax, j, D in zip(axes, combo, mats):
                J[:, ax] = j
                val = val * D[R[:, ax], j]
            full[rows, J @ strides] += coef * val

    for axis in range(d):
        add(-a2diag[:, axis], [axis], [tpl.D2[axis]])
    if cross is not None:
        k = 0
        for a in range(d):
            for b in range(a + 1, d):
                c = -cross[:, k]
                if np.any(c):
                    add(c, [a, b], [tpl.D1[a], tpl.D1[b]])
                k += 1
    if a1 is not None:
        for axis in range(d):
            add(a1[:, axis], [axis], [tpl.D1[axis]])
    if a0 is not None:
        full[rows, R @ strides] += a0
    a_ii = full[:, R @ strides]
    a_ib = full[:, tpl.bnd_all @ strides] @ tpl.Q
    return a_ii, a_ib


def lu_guarded(a_ii):
    """Pivoted dense LU with the reference's relative pivot floor (local_ops.py:422-436)."""
    lu, piv = scipy.linalg.lu_factor(a_ii, check_finite=False)
    diag = np.abs(np.diag(lu))
    dmax = diag.max() if diag.size else 0.0
    singular = bool(diag.size and (dmax == 0.0 or diag.min() <= PIVOT_FLOOR * dmax))
    return (lu, piv), float(diag.min()), float(dmax), singular


def leaf_dtn(tpl, a2diag, a1=None, a0=None, cross=None):
    """DtN map and solution operator of one leaf (local_ops.py:439-446)."""
    a_ii, a_ib = interior_blocks(tpl, a2diag, a1, a0, cross)
    fac, dmin, dmax, singular = lu_guarded(a_ii)
    s = -scipy.linalg.lu_solve(fac, a_ib, check_finite=False)
    dtn = tpl.a_bb + tpl.a_bi @ s
    return dtn, s, (dmin, dmax, singular)


def leaf_reduce_load(tpl, f_int, a2diag, a1=None, a0=None, cross=None):
    """v = A_ii^{-1} f, flux = A_bi v (condensation.py:314-323)."""
    a_ii, _ = interior_blocks(tpl, a2diag, a1, a0, cross)
    fac, dmin, dmax, singular = lu_guarded(a_ii)
    v = scipy.linalg.lu_solve(fac, f_int, check_finite=False)
    return v, tpl.a_bi @ v, (dmin, dmax, singular)


def leaf_interior_solve(tpl, v, ub, a2diag, a1=None, a0=None, cross=None):
    """u_i = v - A_ii^{-1} (A_ib u_b) (condensation.py:379-383)."""
    a_ii, a_ib = interior_blocks(tpl, a2diag, a1, a0, cross)
    fac, dmin, dmax, singular = lu_guarded(a_ii)
    return v - scipy.linalg.lu_solve(fac, a_ib @ ub, check_finite=False), (dmin, dmax, singular)


def dtn_flops(n, m):
    """Dense FLOPs of one leaf reduction as the reference executes it:
    getrf(n) + getrs with m right-hand sides + the m x n x m product."""
    return 2.0 / 3.0 * n ** 3 + 2.0 * n * n * m + 2.0 * n * m * m


# --------------------------------------------------------------------------
# Batched CPU runner (the reference's worker pool, condensation.py:248-264)
# --------------------------------------------------------------------------

def batch_dtn(tpl, coeffs, has_first, has_zeroth, workers=None):
    """DtN maps for a batch: coeffs (B, ncoef, n) packed like the CUDA path."""
    d = tpl.d
    workers = workers or os.cpu_count() or 1

    def one(b):
        c = coeffs[b]
        a2 = c[:d].T
        k = d
        a1 = None
        if has_first:
            a1 = c[k:k + d].T
            k += d
        a0 = c[k] if has_zeroth else None
        return leaf_dtn(tpl, a2, a1, a0)[0]

    if workers == 1:
        return np.stack([one(b) for b in range(coeffs.shape[0])])
    with ThreadPoolExecutor(max_workers=workers) as pool:
        return np.stack(list(pool.map(one, range(coeffs.shape[0]))))


def time_batch_dtn(tpl, coeffs, has_first, has_zeroth, workers=None):
    t0 = time.perf_counter()
    batch_dtn(tpl, coeffs, has_first, has_zeroth, workers)
    return time.perf_counter() - t0
