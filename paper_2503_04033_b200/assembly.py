"""Interface assembly on the device: the leaves' DtN maps scattered into T.

Reference: condensation.py:230-246 (each leaf's T^tau added into the sparse
interface matrix T over its interface DOFs, its Dirichlet columns into the
coupling matrix).  The host mirror (``SparseMatrix`` triplets -> COO -> CSR,
sparse_backend.py) copies every DtN map to the host first; here the maps stay
in HBM and one kernel (``hps_interface_scatter``) adds them into the CSR value
arrays of T and of the coupling C, so only the assembled values cross PCIe.

T is block sparse at face granularity: geometry lays out every face as a
contiguous id range, and a leaf's boundary concatenates its faces
(geometry.py), so the CSR pattern is built from face tables alone — row r of
interface face F holds, in id order, the DOFs of every interface face that
shares a leaf with F — and a scatter job is one (row face, column face) block
of one leaf.  The result is bit-identical to the host path: each entry of T
has at most two contributors and IEEE addition is commutative.
"""

from __future__ import annotations

import ctypes
from itertools import accumulate
from typing import Dict, List, Tuple

import numpy as np
import scipy.sparse as sp

from . import _native
from .errors import ConfigError
from .geometry import Discretization

INTERFACE = "interface"


class InterfacePattern:
    """CSR patterns of T (n_int x n_int) and C (n_int x n_dir) and the per-leaf
    scatter jobs {row0, col0, rows, cols, target, base, stride} (host integers)."""

    def __init__(self, disc: Discretization):
        lo, hi = disc.interface_offset, disc.dirichlet_offset
        self.n_int, self.n_dir = int(disc.n_interface), int(disc.n_dirichlet)
        start: Dict = {}
        size: Dict = {}
        for key, f in disc.faces.items():
            ids = f.node_ids
            if len(ids) and not np.array_equal(ids, np.arange(ids[0], ids[0] + len(ids))):
                raise ConfigError(f"face {key} is not a contiguous id range")
            start[key] = int(ids[0]) - (lo if f.kind == INTERFACE else hi) if len(ids) else 0
            size[key] = len(ids)
        iface = sorted((k for k, f in disc.faces.items() if f.kind == INTERFACE), key=start.get)
        cols: Dict = {}
        row_len = np.zeros((2, len(iface)), dtype=np.int64)
        for i, key in enumerate(iface):
            nb = set()
            for leaf_id in disc.faces[key].leaf_ids:
                if leaf_id is not None:
                    nb.update(disc.leaves[leaf_id].face_keys)
            for t, kind in enumerate((True, False)):
                sel = sorted((g for g in nb if (disc.faces[g].kind == INTERFACE) == kind), key=start.get)
                offs = list(accumulate((size[g] for g in sel), initial=0))
                cols[(t, key)] = dict(zip(sel, offs[:-1]))
                row_len[t, i] = offs[-1]
        sizes = np.asarray([size[k] for k in iface], dtype=np.int64)
        self.indptr, self.indices, base = [], [], []
        for t in range(2):
            per_row = np.repeat(row_len[t], sizes)
            indptr = np.zeros(self.n_int + 1, dtype=np.int64)
            np.cumsum(per_row, out=indptr[1:])
            nnz = int(indptr[-1])
            idx_t = np.int32 if max(nnz, self.n_int, self.n_dir) < 2 ** 31 - 1 else np.int64
            indices = np.empty(nnz, dtype=idx_t)
            bases = indptr[[start[key] for key in iface]].tolist() if iface else []
            for key, b0 in zip(iface, bases):  # rows of a face share one column list: broadcast it
                sel = cols[(t, key)]
                if not sel:
                    continue
                row = np.concatenate([np.arange(start[g], start[g] + size[g]) for g in sel])
                indices[b0:b0 + size[key] * len(row)].reshape(size[key], len(row))[:] = row
            self.indices.append(indices)
            self.indptr.append(indptr.astype(idx_t))
            base.append(dict(zip(iface, bases)))
        self.nnz = (int(self.indptr[0][-1]), int(self.indptr[1][-1]))
        # the index arrays are shared by every T / C built from this (cached) pattern:
        # read-only, so an in-place edit of a returned matrix (eliminate_zeros, prune,
        # sort_indices) raises instead of corrupting later builds of the same mesh
        for a in self.indptr + self.indices:
            a.flags.writeable = False
        pos = {k: i for i, k in enumerate(iface)}
        self.leaf_jobs: List[np.ndarray] = []
        for leaf in disc.leaves:
            jobs = []
            offs = list(accumulate((size[k] for k in leaf.face_keys), initial=0))
            for fi, fk in enumerate(leaf.face_keys):
                if disc.faces[fk].kind != INTERFACE:
                    continue
                for gi, gk in enumerate(leaf.face_keys):
                    t = 0 if disc.faces[gk].kind == INTERFACE else 1
                    stride = int(row_len[t, pos[fk]])
                    jobs.append((offs[fi], offs[gi], size[fk], size[gk], t,
                                 base[t][fk] + cols[(t, fk)][gk], stride))
            self.leaf_jobs.append(np.asarray(jobs, dtype=np.int64).reshape(-1, 7))
        # vector jobs (interface fluxes into g_b): one column per interface face
        self.leaf_vec_jobs = [
            np.asarray([(offs_l[fi], 0, size[fk], 1, 0, start[fk], 1)
                        for fi, fk in enumerate(leaf.face_keys) if disc.faces[fk].kind == INTERFACE],
                       dtype=np.int64).reshape(-1, 7)
            for leaf in disc.leaves
            for offs_l in [list(accumulate((size[k] for k in leaf.face_keys), initial=0))]]
        self.job_offsets, self.all_jobs = self._table(self.leaf_jobs)
        self.vec_offsets, self.all_vec_jobs = self._table(self.leaf_vec_jobs)

    @staticmethod
    def _table(leaf_jobs):
        """Every leaf's jobs with its global leaf id in column 0, and per-leaf row offsets."""
        counts = [len(j) for j in leaf_jobs]
        offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        table = np.concatenate(
            [np.repeat(np.arange(len(counts), dtype=np.int64), counts)[:, None],
             np.concatenate(leaf_jobs) if counts else np.empty((0, 7), np.int64)], axis=1)
        return offsets, table

    def jobs_for(self, ids, vectors: bool = False) -> np.ndarray:
        """int64 [jobs][8] for a flush of leaves ids (column 0 = position in the flush)."""
        source = self.leaf_vec_jobs if vectors else self.leaf_jobs
        parts = []
        for k, leaf_id in enumerate(ids):
            j = source[leaf_id]
            parts.append(np.concatenate([np.full((len(j), 1), k, dtype=np.int64), j], axis=1))
        return np.ascontiguousarray(np.concatenate(parts) if parts else np.empty((0, 8), np.int64))

    def matrices(self, t_vals: np.ndarray, c_vals: np.ndarray) -> Tuple[sp.csr_matrix, sp.csr_matrix]:
        t = sp.csr_matrix((t_vals, self.indices[0], self.indptr[0]), shape=(self.n_int, self.n_int))
        c = sp.csr_matrix((c_vals, self.indices[1], self.indptr[1]), shape=(self.n_int, self.n_dir))
        t.has_sorted_indices = True
        c.has_sorted_indices = True
        return t, c


def pattern_for(disc: Discretization) -> InterfacePattern:
    """The mesh's pattern, built once per discretization (it depends only on
    the face and leaf tables, which never change after construction)."""
    pat = getattr(disc, "_interface_pattern", None)
    if pat is None:
        pat = InterfacePattern(disc)
        disc._interface_pattern = pat
    return pat


class DeviceAssembler:
    """Accumulates flushes of device DtN maps into device CSR values of T and C
    (or, with ``vectors=True``, interface fluxes into the interface RHS)."""

    def __init__(self, pattern: InterfacePattern, device: int, vectors: bool = False):
        import torch
        self.torch, self.pattern, self.device = torch, pattern, int(device)
        dev = f"cuda:{self.device}"
        self.lib = _native.load()
        if vectors:
            self.g = torch.zeros(max(pattern.n_int, 1), dtype=torch.float64, device=dev)
            table, self.offsets = pattern.all_vec_jobs, pattern.vec_offsets
        else:
            self.t_vals = torch.zeros(max(pattern.nnz[0], 1), dtype=torch.float64, device=dev)
            self.c_vals = torch.zeros(max(pattern.nnz[1], 1), dtype=torch.float64, device=dev)
            table, self.offsets = pattern.all_jobs, pattern.job_offsets
        self.vectors = vectors
        self.jobs = torch.from_numpy(np.ascontiguousarray(table)).to(dev)  # uploaded once
        self._keep = None  # the last flush's inputs / job table, alive until the kernel is ordered

    def _launch(self, blocks, ld: int, block_stride: int, ids, out0, out1) -> None:
        torch = self.torch
        ids = list(ids)
        if not ids:
            return
        off = self.offsets
        if ids == list(range(ids[0], ids[0] + len(ids))):  # a contiguous flush: the resident table
            lo, hi = int(off[ids[0]]), int(off[ids[-1] + 1])
            jobs, n_jobs, leaf0 = self.jobs[lo:hi], hi - lo, ids[0]
        else:
            jobs_h = self.pattern.jobs_for(ids, vectors=self.vectors)
            jobs = torch.from_numpy(jobs_h).to(f"cuda:{self.device}")
            n_jobs, leaf0 = len(jobs_h), 0
        if n_jobs == 0:
            return
        # torch's current stream: the caller's launch stream, the one the maps were
        # produced on and the one finish() reads the values after
        s = torch.cuda.current_stream(self.device)
        _native.check(self.lib.hps_interface_scatter(
            self.device, ctypes.c_void_p(blocks.data_ptr()), ld, block_stride, leaf0, n_jobs,
            ctypes.c_void_p(jobs.data_ptr()), ctypes.c_void_p(out0.data_ptr()),
            ctypes.c_void_p(out1.data_ptr()), ctypes.c_void_p(s.cuda_stream)))
        self._keep = (blocks, jobs)

    def add(self, dtn, ids) -> None:
        """Scatter-add the DtN maps of a flush (device tensor [len(ids)][m][m])."""
        if self.vectors:
            raise ConfigError("this assembler accumulates interface vectors")
        if dtn.dim() != 3 or dtn.shape[0] != len(ids) or dtn.shape[1] != dtn.shape[2]:
            raise ConfigError(f"DtN batch of shape {tuple(dtn.shape)} for {len(ids)} leaves")
        dtn = dtn.contiguous()
        m = int(dtn.shape[1])
        self._launch(dtn, m, m * m, ids, self.t_vals, self.c_vals)

    def add_vectors(self, flux, ids) -> None:
        """Add the interface part of per-leaf boundary vectors (device [len(ids)][m])."""
        if not self.vectors:
            raise ConfigError("this assembler accumulates T and C")
        if flux.dim() != 2 or flux.shape[0] != len(ids):
            raise ConfigError(f"flux batch of shape {tuple(flux.shape)} for {len(ids)} leaves")
        flux = flux.contiguous()
        self._launch(flux, 1, int(flux.shape[1]), ids, self.g, self.g)

    def finish(self) -> Tuple[sp.csr_matrix, sp.csr_matrix]:
        nt, nc = self.pattern.nnz
        t_vals = self.t_vals[:nt].cpu().numpy()   # synchronizes the current stream
        c_vals = self.c_vals[:nc].cpu().numpy()
        self._keep = None
        return self.pattern.matrices(t_vals, c_vals)

    def finish_vector(self) -> np.ndarray:
        g = self.g[:self.pattern.n_int].cpu().numpy()
        self._keep = None
        return g
