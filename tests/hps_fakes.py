"""CPU stand-ins for the rank's GPU in multi-process gloo tests (TEST ONLY).

``OracleEngine`` has the LeafEngine methods the solver stages call, computing
each leaf with the CPU oracle; ``ReplayAssembler`` replays the jobs of
``hps_interface_scatter`` with numpy.  ``install()`` swaps them into the
condensation module of the current process, so the stages' sharding, flush
and collective logic runs unchanged on CPU tensors over gloo.
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import hps_oracle as O


class OracleEngine:
    def __init__(self, template, coeffs, slots: int = 3):
        self.tpl = O.OracleTemplate(template.widths, template.p, template.corner_mode)
        self.d = template.d
        self.n, self.m = template.n_interior, template.n_boundary
        self.has_first = coeffs.first_order is not None
        self.has_zeroth = coeffs.zeroth_order is not None
        self.ncoef = self.d + (self.d if self.has_first else 0) + (1 if self.has_zeroth else 0)
        self.slots = slots
        self.device = "cpu"
        self.launches = 0

    # layout of include/hps_leaf.h: diagonal second order, first order, zeroth
    def _unpack(self, c):
        d = self.d
        a1 = c[d:2 * d].T if self.has_first else None
        a0 = c[-1] if self.has_zeroth else None
        return c[:d].T, a1, a0

    def empty(self, *shape):
        return torch.empty(shape, dtype=torch.float64)

    def stage(self, pack):
        return torch.from_numpy(np.ascontiguousarray(pack, dtype=np.float64))

    def synchronize(self):
        pass

    def workspace(self):
        return 0, 0

    def dtn(self, coeffs, out=None, stats=None, stream=None):
        pack = coeffs.numpy()
        L = pack.shape[0]
        out = self.empty(L, self.m, self.m) if out is None else out
        stats = self.empty(L, 2) if stats is None else stats
        self.launches += 1
        for k in range(L):
            t, _, (dmin, dmax, _) = O.leaf_dtn(self.tpl, *self._unpack(pack[k]))
            out[k] = torch.from_numpy(t)
            stats[k, 0], stats[k, 1] = dmin, dmax
        return out, stats

    def dtn_host(self, pack):
        out, stats = self.dtn(self.stage(pack))
        return out.numpy(), stats.numpy()

    def reduce_load(self, coeffs, f):
        pack = coeffs.numpy()
        f = np.asarray(f, dtype=np.float64)
        L = pack.shape[0]
        v, flux, stats = self.empty(L, self.n), self.empty(L, self.m), self.empty(L, 2)
        self.launches += 1
        for k in range(L):
            vk, fk, (dmin, dmax, _) = O.leaf_reduce_load(self.tpl, f[k], *self._unpack(pack[k]))
            v[k], flux[k] = torch.from_numpy(vk), torch.from_numpy(fk)
            stats[k, 0], stats[k, 1] = dmin, dmax
        return v, flux, stats

    def reduce_load_host(self, pack, f):
        v, flux, stats = self.reduce_load(self.stage(pack), f)
        return v.numpy(), flux.numpy(), stats.numpy()

    def interior_solve_host(self, pack, ub, v):
        L = pack.shape[0]
        u, stats = np.empty((L, self.n)), np.empty((L, 2))
        self.launches += 1
        for k in range(L):
            u[k], (dmin, dmax, _) = O.leaf_interior_solve(self.tpl, v[k], ub[k], *self._unpack(pack[k]))
            stats[k] = dmin, dmax
        return u, stats


class ReplayAssembler:
    """numpy replay of hps_interface_scatter over InterfacePattern.jobs_for."""

    def __init__(self, pattern, device, vectors: bool = False):
        self.pattern, self.vectors = pattern, vectors
        if vectors:
            self.g = torch.zeros(max(pattern.n_int, 1), dtype=torch.float64)
        else:
            self.t_vals = torch.zeros(max(pattern.nnz[0], 1), dtype=torch.float64)
            self.c_vals = torch.zeros(max(pattern.nnz[1], 1), dtype=torch.float64)

    def _replay(self, blocks, ids, outs, vectors):
        for k, r0, c0, nr, nc, tgt, base, stride in self.pattern.jobs_for(ids, vectors=vectors):
            blk = blocks[k, r0:r0 + nr, c0:c0 + nc] if not vectors else blocks[k, r0:r0 + nr, None]
            idx = base + np.arange(nr)[:, None] * stride + np.arange(nc)[None, :]
            np.add.at(outs[tgt], idx, blk)

    def add(self, dtn, ids, stream=None):
        self._replay(dtn.numpy(), list(ids), [self.t_vals.numpy(), self.c_vals.numpy()], False)

    def add_vectors(self, flux, ids, stream=None):
        g = self.g.numpy()
        self._replay(flux.numpy(), list(ids), [g, g], True)

    def finish(self):
        nt, nc = self.pattern.nnz
        return self.pattern.matrices(self.t_vals[:nt].numpy().copy(), self.c_vals[:nc].numpy().copy())

    def finish_vector(self):
        return self.g[:self.pattern.n_int].numpy().copy()


def install(slots: int = 3):
    """Route the condensation stages of this process through the CPU stand-ins;
    returns the list of engines created (for launch counting)."""
    from paper_2503_04033_b200 import condensation
    made = []

    def engine_for(template, coeffs, resolved):
        eng = OracleEngine(template, coeffs, slots=slots)
        made.append(eng)
        return eng

    condensation._engine_for = engine_for
    condensation.DeviceAssembler = ReplayAssembler
    return made
