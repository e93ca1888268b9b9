"""GPU leaf engine: the Python face of libhps_leaf.so.

A :class:`LeafEngine` wraps one device plan (templates uploaded once, a slot
workspace per SM) and exposes the batched leaf operations of the two-level
solver on device tensors (torch, CUDA) or host arrays (numpy):

=========================  ==============================================
``dtn``                    T^tau = A_bb - A_bi A_ii^{-1} A_ib  (build stage)
``solution_operator``      S^tau = -A_ii^{-1} A_ib
``reduce_load``            v = A_ii^{-1} f,  flux = A_bi v
``interior_solve``         u_i = v - A_ii^{-1} (A_ib u_b)
=========================  ==============================================

PyTorch only supplies device memory and streams; the arithmetic is in the
CUDA kernels.  There is no CPU fallback: without a CUDA device or the built
library every call raises :class:`NativeUnavailableError`.
"""

from __future__ import annotations

import os

import ctypes
import functools
from typing import Optional, Tuple

import numpy as np

from . import _native
from .errors import ConfigError, NativeUnavailableError
from .local_ops import DROP_CORNERS, LEGENDRE_FACES, LeafTemplate, coefficient_layout


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailableError("a CUDA device is required: the leaf path has no CPU fallback")
    return torch


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


def _np_ptr(a: Optional[np.ndarray]) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data if a is not None else 0)


class LeafEngine:
    """One device plan for equal leaves of a mesh (shape, order, coefficient layout).

    A plan's slot workspace (tens of GB at p >= 16) is allocated by its first
    launch and held until :meth:`release` — ``for_template`` keeps a small cache of
    plans and releases the workspace of every other cached plan on the device
    before handing one out, so only the plan in use holds device memory.
    """

    _plans = {}
    MAX_CACHED = 4

    def __init__(self, template: LeafTemplate, has_first: bool, has_zeroth: bool,
                 device: int = 0, max_slots: int = 0, workspace_budget: int = 0,
                 has_cross: bool = False):
        if has_cross and template.corner_mode != LEGENDRE_FACES:
            raise ConfigError("cross-derivative terms require legendre face grids")
        self.lib = _native.load()
        torch = _torch()
        self.torch = torch
        self.device = int(device)
        self.template = template
        self.d, self.p = template.d, template.p
        self.n, self.m = template.n_interior, template.n_boundary
        self.has_first, self.has_zeroth = bool(has_first), bool(has_zeroth)
        self.has_cross = bool(has_cross)
        self.legendre = template.corner_mode == LEGENDRE_FACES
        self.ncoef = (self.d + (self.d * (self.d - 1) // 2 if has_cross else 0)
                      + (self.d if has_first else 0) + (1 if has_zeroth else 0))
        D1 = np.ascontiguousarray(np.stack(template.diff))
        D2 = np.ascontiguousarray(np.stack(template.diff2))
        a_bi = np.ascontiguousarray(template.a_bi)
        a_bb = np.ascontiguousarray(template.a_bb)
        plan = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            if self.legendre:
                Q = np.ascontiguousarray(template._boundary_injection)
                bpos = np.full(template.n_grid, -1, dtype=np.int32)
                bpos[template.boundary_all_idx] = np.arange(template.boundary_all_idx.size,
                                                            dtype=np.int32)
                _native.check(self.lib.hps_plan_create_legendre(
                    ctypes.byref(plan), self.device, self.d, self.p, int(has_cross),
                    int(has_first), int(has_zeroth), _np_ptr(D1), _np_ptr(D2), _np_ptr(a_bi),
                    _np_ptr(a_bb), _np_ptr(Q), int(Q.shape[0]), _np_ptr(bpos), int(max_slots),
                    int(workspace_budget)))
            else:
                _native.check(self.lib.hps_plan_create(
                    ctypes.byref(plan), self.device, self.d, self.p, int(has_first),
                    int(has_zeroth), _np_ptr(D1), _np_ptr(D2), _np_ptr(a_bi), _np_ptr(a_bb),
                    int(max_slots), int(workspace_budget)))
        self.plan = plan
        n, m, nc, slots = (ctypes.c_int() for _ in range(4))
        dtn_b, sol_b = ctypes.c_size_t(), ctypes.c_size_t()
        _native.check(self.lib.hps_plan_info(plan, ctypes.byref(n), ctypes.byref(m), ctypes.byref(nc),
                                             ctypes.byref(slots), ctypes.byref(dtn_b),
                                             ctypes.byref(sol_b)))
        assert n.value == self.n and m.value == self.m and nc.value == self.ncoef
        self.slots = slots.value
        self.dtn_slot_bytes = dtn_b.value
        self.solve_slot_bytes = sol_b.value

    def __del__(self):
        plan = getattr(self, "plan", None)
        if plan is not None and plan.value:
            try:
                self.lib.hps_plan_destroy(plan)
            except Exception:
                pass
            self.plan = None

    @classmethod
    def for_template(cls, template: LeafTemplate, coeffs, device: int = 0, **kw) -> "LeafEngine":
        has_first, has_zeroth, has_cross = coefficient_layout(coeffs)
        key = (tuple(float(w) for w in template.widths), template.p, template.corner_mode, has_first,
               has_zeroth, has_cross, int(device), tuple(sorted(kw.items())))
        eng = cls._plans.pop(key, None)
        for other in cls._plans.values():        # one workspace per device at a time
            if other.device == int(device):
                other.release()
        if eng is None:
            while len(cls._plans) >= cls.MAX_CACHED:   # drop the least recently used: its
                cls._plans.pop(next(iter(cls._plans))).release()  # plan dies with its last user
            eng = cls(template, has_first, has_zeroth, device=device, has_cross=has_cross, **kw)
        cls._plans[key] = eng                   # most recently used last
        return eng

    @classmethod
    def clear_cache(cls) -> None:
        """Drop every cached plan and free its workspace."""
        while cls._plans:
            cls._plans.popitem()[1].release()

    def release(self) -> None:
        """Free the slot workspace and streaming buffers (after the last launch
        finishes); the next call re-allocates them."""
        bufs = getattr(self, "_stage_bufs", None)
        if bufs is not None:
            for b in bufs:
                if b is not None:
                    b[2].synchronize()
            self._stage_bufs = None
        if self.plan is not None and self.plan.value:
            _native.check(self.lib.hps_plan_release(self.plan))

    def close(self) -> None:
        self.__del__()

    def workspace(self) -> Tuple[int, int]:
        """(device bytes held now, slots they are sized for)."""
        b, s = ctypes.c_size_t(), ctypes.c_int()
        _native.check(self.lib.hps_plan_workspace(self.plan, ctypes.byref(b), ctypes.byref(s)))
        return int(b.value), int(s.value)

    # ---------------------------------------------------------------- helpers
    def _stream(self, stream):
        torch = self.torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(s.cuda_stream)

    def _check_coeffs(self, coeffs):
        if tuple(coeffs.shape[1:]) != (self.ncoef, self.n):
            raise ConfigError(f"coefficient pack has shape {tuple(coeffs.shape)}, "
                              f"expected (leaves, {self.ncoef}, {self.n})")

    def _dev(self, a):
        torch = self.torch
        if isinstance(a, torch.Tensor):
            return a.to(device=f"cuda:{self.device}", dtype=torch.float64).contiguous()
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(f"cuda:{self.device}")

    def _empty(self, *shape):
        return self.torch.empty(shape, dtype=self.torch.float64, device=f"cuda:{self.device}")

    empty = _empty

    def synchronize(self) -> None:
        self.torch.cuda.synchronize(self.device)

    def stage(self, pack: np.ndarray, stream=None):
        """Host coefficient pack -> device tensor through a pinned double buffer: the
        H2D copy is queued on the launch stream and the host returns at once (it
        packs the next flush while the device works on this one)."""
        torch = self.torch
        pack = np.ascontiguousarray(pack, dtype=np.float64)
        self._check_coeffs(pack)
        L = pack.shape[0]
        self._stage_k = (getattr(self, "_stage_k", 0) + 1) % 2
        bufs = getattr(self, "_stage_bufs", None)
        if bufs is None:
            bufs = self._stage_bufs = [None, None]
        b = bufs[self._stage_k]
        if b is None or b[0].shape[0] < L:
            if b is not None:
                b[2].synchronize()
            shape = (L, self.ncoef, self.n)
            b = bufs[self._stage_k] = (torch.empty(shape, dtype=torch.float64, pin_memory=True),
                                       self._empty(*shape), torch.cuda.Event())
        host, dev, done = b
        done.synchronize()                       # the last copy out of this host buffer is over
        host[:L].numpy()[:] = pack
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(s):
            dev[:L].copy_(host[:L], non_blocking=True)
            done.record(s)
        return dev[:L]

    # ---------------------------------------------------------- device calls
    def dtn(self, coeffs, out=None, stats=None, stream=None):
        """DtN maps (leaves, m, m) for device coefficient packs (leaves, ncoef, n)."""
        coeffs = self._dev(coeffs)
        self._check_coeffs(coeffs)
        L = coeffs.shape[0]
        out = self._empty(L, self.m, self.m) if out is None else out
        stats = self._empty(L, 2) if stats is None else stats
        _native.check(self.lib.hps_leaf_dtn(self.plan, L, _ptr(coeffs), _ptr(out), _ptr(stats),
                                            self._stream(stream)))
        return out, stats

    def factors(self, coeffs, stream=None):
        """DtN maps (leaves, m, m) and solution operators (leaves, n, m) from one
        factorization per leaf (one launch)."""
        coeffs = self._dev(coeffs)
        self._check_coeffs(coeffs)
        L = coeffs.shape[0]
        dtn, s, stats = self._empty(L, self.m, self.m), self._empty(L, self.n, self.m), self._empty(L, 2)
        _native.check(self.lib.hps_leaf_factors(self.plan, L, _ptr(coeffs), _ptr(dtn), _ptr(s),
                                                _ptr(stats), self._stream(stream)))
        return dtn, s, stats

    def solution_operator(self, coeffs, stream=None):
        coeffs = self._dev(coeffs)
        self._check_coeffs(coeffs)
        L = coeffs.shape[0]
        s, stats = self._empty(L, self.n, self.m), self._empty(L, 2)
        _native.check(self.lib.hps_leaf_solution_operator(self.plan, L, _ptr(coeffs), _ptr(s),
                                                          _ptr(stats), self._stream(stream)))
        return s, stats

    def reduce_load(self, coeffs, f, stream=None):
        coeffs, f = self._dev(coeffs), self._dev(f)
        self._check_coeffs(coeffs)
        L = coeffs.shape[0]
        v, flux, stats = self._empty(L, self.n), self._empty(L, self.m), self._empty(L, 2)
        _native.check(self.lib.hps_leaf_reduce_load(self.plan, L, _ptr(coeffs), _ptr(f), _ptr(v),
                                                     _ptr(flux), _ptr(stats), self._stream(stream)))
        return v, flux, stats

    def interior_solve(self, coeffs, ub, v, stream=None):
        coeffs, ub, v = self._dev(coeffs), self._dev(ub), self._dev(v)
        self._check_coeffs(coeffs)
        L = coeffs.shape[0]
        u, stats = self._empty(L, self.n), self._empty(L, 2)
        _native.check(self.lib.hps_leaf_interior_solve(self.plan, L, _ptr(coeffs), _ptr(ub), _ptr(v),
                                                       _ptr(u), _ptr(stats), self._stream(stream)))
        return u, stats

    def apply(self, coeffs, u_int, u_b, stream=None):
        """w = collocation rows applied to [u_int; u_b] per leaf (drop plans)."""
        coeffs, u_int, u_b = self._dev(coeffs), self._dev(u_int), self._dev(u_b)
        self._check_coeffs(coeffs)
        L = coeffs.shape[0]
        w = self._empty(L, self.n)
        _native.check(self.lib.hps_leaf_apply(self.plan, L, _ptr(coeffs), _ptr(u_int), _ptr(u_b),
                                              _ptr(w), self._stream(stream)))
        return w

    # ------------------------------------------------------------ host calls
    def dtn_host(self, coeffs: np.ndarray, out: Optional[np.ndarray] = None,
                 chunk_leaves: int = 0) -> Tuple[np.ndarray, np.ndarray]:
        """Host-buffer DtN through the streamed C entry (H2D / kernel / D2H overlap)."""
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        self._check_coeffs(coeffs)
        L = coeffs.shape[0]
        if out is None:
            out = np.empty((L, self.m, self.m))
        stats = np.empty((L, 2))
        _native.check(self.lib.hps_leaf_dtn_host(self.plan, L, _np_ptr(coeffs), _np_ptr(out),
                                                 _np_ptr(stats), int(chunk_leaves)))
        return out, stats

    def factors_host(self, coeffs):
        dtn, s, stats = self.factors(coeffs)
        return dtn.cpu().numpy(), s.cpu().numpy(), stats.cpu().numpy()

    def apply_host(self, coeffs, u_int, u_b):
        return self.apply(coeffs, u_int, u_b).cpu().numpy()

    def solution_operator_host(self, coeffs):
        s, stats = self.solution_operator(coeffs)
        return s.cpu().numpy(), stats.cpu().numpy()

    def reduce_load_host(self, coeffs, f):
        v, flux, stats = self.reduce_load(coeffs, f)
        return v.cpu().numpy(), flux.cpu().numpy(), stats.cpu().numpy()

    def interior_solve_host(self, coeffs, ub, v):
        u, stats = self.interior_solve(coeffs, ub, v)
        return u.cpu().numpy(), stats.cpu().numpy()


def dtn_flops(n: int, m: int) -> float:
    """FLOPs of one leaf reduction in the reference's dense algorithm:
    getrf(n) + getrs with m right-hand sides + the (m x n) @ (n x m) product."""
    return 2.0 / 3.0 * n ** 3 + 2.0 * n * n * m + 2.0 * n * m * m


def _first_nonzero(rowpos: np.ndarray, q: int, d: int) -> np.ndarray:
    """g[v]: smallest slot position among the nodes on v's d grid lines."""
    pos = rowpos.reshape((q,) * d)
    mins = [pos.min(axis=a, keepdims=True) for a in range(d)]
    g = mins[0]
    for mn in mins[1:]:
        g = np.minimum(g, mn)
    return np.broadcast_to(g, (q,) * d).reshape(-1).copy()


def interior_order(q: int, d: int = 3, natural: bool = False) -> np.ndarray:
    """Slot position of every natural interior node in the DtN drop mode (mirror
    of build_orderings in hps_leaf.cu): growing cubes from a leaf corner (shell =
    max coordinate), within a shell by the first nonzero g under the plain
    shell order, then the natural index."""
    n = q ** d
    idx = np.arange(n)
    if natural:
        return idx
    I = np.stack(np.unravel_index(idx, (q,) * d), axis=1)
    shell = I.max(axis=1)
    corner = np.empty(n, dtype=np.int64)
    corner[np.lexsort((idx, shell))] = np.arange(n)
    g = _first_nonzero(corner, q, d)
    rowpos = np.empty(n, dtype=np.int64)
    rowpos[np.lexsort((idx, g, shell))] = np.arange(n)
    return rowpos


def forward_prefix_rows(q: int, d: int = 3, natural: bool = False) -> np.ndarray:
    """First slot row of every boundary DOF's line (the zero prefix of its A_ib
    column that the forward solve skips), natural face order."""
    rowpos = interior_order(q, d, natural)
    if d == 3:
        t = np.arange(q * q)
        bases = [(t, q * q), ((t // q) * q * q + t % q, q), (t * q, 1)]
    else:
        t = np.arange(q)
        bases = [(t, q), (t * q, 1)]
    f = []
    for base, stride in bases:
        rows = base[:, None] + stride * np.arange(q)[None, :]
        fa = rowpos[rows].min(axis=1)
        f += [fa, fa]
    return np.concatenate(f)


@functools.lru_cache(maxsize=None)
def leaf_work_model(q: int, d: int = 3) -> dict:
    """Work of the engine's DtN op program for one leaf, by phase (drop mode,
    engine orderings, no interchanges — 10% of the pivots, which move rows
    together with their first-nonzero entry).  Mirrors the program builder:
    every 32 x 32 warp block of a GEMM tile starts its k loop at the first
    nonzero of its rows (16-row group minima), of its trailing LU columns
    (first row of U with a nonzero) and of its RHS columns, in k chunks of 16
    (8 on the 256 x 32 tiles), and is skipped when that lies beyond the k range;
    triangular base blocks count h^2 per column; narrow panels rows * w^2."""
    n = q ** d
    n_pad = (n + 15) // 16 * 16
    rowpos = interior_order(q, d)
    g = _first_nonzero(rowpos, q, d)
    gpos = np.arange(n_pad)
    gpos[rowpos] = g
    g16 = np.array([gpos[i:i + 16].min() for i in range(0, n_pad, 16)])
    fs = np.sort(forward_prefix_rows(q, d))          # RHS columns in slot order
    m = fs.size
    TN = 128

    def split16(w):
        if w > 2 * TN:
            h = (w // 2) // TN * TN
            return TN if h < TN else h
        return ((w // 2 + 15) // 16) * 16

    def sub(r0, M, k0, K, ncols, col_first=None):
        """sum over the 32 x 32 warp blocks of every tile of 2 rows cols k_eff: each
        warp starts at the first k chunk its own rows (16-row minima of g) and
        columns (col_first, per column) need, chunk KC = 16 (64 x 128 tiles) or
        8 (256 x 32 tiles for N <= 64), as the kernel's per-warp bounds"""
        if M <= 0 or K <= 0 or ncols <= 0:
            return 0.0
        kc = 8 if (ncols <= 64 and M >= 256) else 16
        tot = 0.0
        for tr in range(r0, r0 + M, 32):
            rows = min(32, r0 + M - tr)
            kr = g16[tr // 16:(tr + rows + 15) // 16].min() - k0
            for tc in range(0, ncols, 32):
                cols = min(32, ncols - tc)
                kk = kr if col_first is None else max(kr, col_first[tc:tc + cols].min() - k0)
                if kk >= K:
                    continue
                kk = max(kk, 0) // kc * kc
                tot += 2.0 * rows * cols * (K - kk)
        return tot

    work = {"panel": 0.0, "lu_trsm": 0.0, "lu_update": 0.0, "forward": 0.0}

    def trsm_lower(r0, h, ncols, key, col_first=None, ncl=None):
        if h <= 64:
            nc = ncols if ncl is None else ncl(r0 + h)
            work[key] += float(h) * h * nc
            return
        h1 = split16(h)
        trsm_lower(r0, h1, ncols, key, col_first, ncl)
        nc = ncols if ncl is None else ncl(r0 + h1)
        work[key] += sub(r0 + h1, h - h1, r0, h1, nc, col_first)
        trsm_lower(r0 + h1, h - h1, ncols, key, col_first, ncl)

    def lu(c0, w):
        if w <= 32:
            work["panel"] += float(n_pad - c0) * w * w
            return
        h = split16(w)
        lu(c0, h)
        # trailing columns start at their first nonzero row of U (symmetric pattern:
        # g of the column's node), valid up to the first interchange
        cf = gpos[c0 + h:c0 + w]
        trsm_lower(c0, h, w - h, "lu_trsm", cf)
        work["lu_update"] += sub(c0 + h, n_pad - c0 - h, c0, h, w - h, cf)
        lu(c0 + h, w - h)

    lu(0, n_pad)
    trsm_lower(0, n_pad, m, "forward", fs, lambda R: int(np.searchsorted(fs, R, side="left")))
    j = np.arange(m)
    f = fs.astype(float)
    # W = A_bi U^-1: row b from its first nonzero f_b; column c of U from its first
    # nonzero row (16-column minima of g, as the kernel's column bounds)
    gc = np.repeat(g16, 16)[:n]
    cols = np.arange(n)
    work["W"] = float(sum(2.0 * np.maximum(cols[fb:] - np.maximum(fb, gc[fb:]), 0).sum()
                          for fb in fs))
    work["T"] = 2.0 * float(((2 * j + 1) * (n - f)).sum())
    return work


def dtn_flops_executed(n: int, m: int, q: int, d: int = 3, skip_prefix: bool = True,
                       wtrick: bool = True) -> float:
    """FLOPs of the algorithm the engine runs for one leaf (drop mode): the LU
    and the forward solve Y = L^-1 P A_ib with their structurally zero tiles
    skipped (leaf_work_model: rows from their first nonzero, RHS columns from
    their line's first row), and then either
      wtrick:  W = A_bi U^-1 from each row's first nonzero and each column's first
               row of U (sum over j >= f_b of 2 (j - max(f_b, g_j))) and
               T -= W Y over k >= max(f_b, f_c) (sum 2 (n - max(f_b, f_c)));
      else:    the backward solve (n^2 m) and the line-sparse A_bi X (2 q m^2).
    f from the engine's interior order (forward_prefix_rows).  skip_prefix=False:
    the dense variant 2/3 n^3 + 2 n^2 m + 2 q m^2 (legendre faces)."""
    if not skip_prefix:
        return 2.0 / 3.0 * n ** 3 + 2.0 * n * n * m + 2.0 * q * m * m
    w = leaf_work_model(q, d)
    lu_fwd = w["panel"] + w["lu_trsm"] + w["lu_update"] + w["forward"]
    if (n + 15) // 16 * 16 < int(os.environ.get("HPS_WT_MIN_N", "1536")):
        wtrick = False               # the engine uses W blocks from n_pad >= 1536 (p >= 14) on
    if not wtrick:
        return lu_fwd + float(n) * n * m + 2.0 * q * m * m
    return lu_fwd + w["W"] + w["T"]
