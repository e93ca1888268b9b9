"""Device interface assembly (assembly.py) against the reference's host scatter
(condensation.py:230-246 -> scatter_leaf_blocks / finalize_host).

CPU tests replay the kernel's scatter jobs with numpy on random DtN maps; the
GPU tests run hps_interface_scatter and whole builds through both paths.  The
bar is bit-exact: same CSR structure, same values."""

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2503_04033_b200.assembly import InterfacePattern
from paper_2503_04033_b200.condensation import (_make_dof_map, finalize_host,
                                                scatter_leaf_blocks)
from paper_2503_04033_b200.geometry import DomainBox, MeshConfig, build_discretization
from paper_2503_04033_b200.local_ops import LeafTemplate
from paper_2503_04033_b200.sparse_backend import SparseMatrix

CASES = [((1, 1), 6, "drop"), ((3, 2), 6, "drop"), ((2, 2), 5, "legendre"),
         ((1, 1, 1), 5, "drop"), ((2, 1, 1), 5, "drop"), ((3, 2, 2), 6, "drop"),
         ((2, 2, 2), 5, "legendre")]


def _disc(boxes, p, mode):
    d = len(boxes)
    return build_discretization(DomainBox((0.0,) * d, (1.0,) * d), MeshConfig(boxes, p, mode))


def _host(disc, dtn):
    tpl = LeafTemplate(disc.leaf_widths, disc.p, disc.corner_mode, False)
    dof_map = _make_dof_map(disc, tpl)
    tb, cr, cc, cv = SparseMatrix(disc.n_interface), [], [], []
    scatter_leaf_blocks(dof_map, range(len(disc.leaves)), dtn, tb, cr, cc, cv)
    return finalize_host(tb, cr, cc, cv, disc.n_interface, disc.n_dirichlet)


def _replay(pat, dtn, ids):
    """numpy replay of hps_interface_scatter_kernel over jobs_for(ids)."""
    out = [np.zeros(pat.nnz[0]), np.zeros(pat.nnz[1])]
    for k, r0, c0, nr, nc, tgt, base, stride in pat.jobs_for(ids):
        blk = dtn[k, r0:r0 + nr, c0:c0 + nc]
        idx = base + np.arange(nr)[:, None] * stride + np.arange(nc)[None, :]
        np.add.at(out[tgt], idx, blk)
    return out


def _same(a, b):
    a, b = sp.csr_matrix(a), sp.csr_matrix(b)
    assert a.shape == b.shape
    assert np.array_equal(a.indptr, b.indptr)
    assert np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.data, b.data)  # bit-exact (no tolerance)


@pytest.mark.parametrize("boxes,p,mode", CASES)
def test_pattern_and_jobs_reproduce_host_scatter(boxes, p, mode):
    disc = _disc(boxes, p, mode)
    m = len(disc.leaves[0].boundary_ids)
    rng = np.random.default_rng(len(disc.leaves) * 31 + p)
    dtn = rng.standard_normal((len(disc.leaves), m, m))
    t_ref, c_ref = _host(disc, dtn)
    pat = InterfacePattern(disc)
    ids = list(range(len(disc.leaves)))
    t_vals, c_vals = _replay(pat, dtn, ids)
    t, c = pat.matrices(t_vals, c_vals)
    _same(t, t_ref)
    _same(c, c_ref)


def test_flushes_in_any_order_give_the_same_values():
    disc = _disc((3, 2, 2), 5, "drop")
    m = len(disc.leaves[0].boundary_ids)
    dtn = np.random.default_rng(3).standard_normal((len(disc.leaves), m, m))
    pat = InterfacePattern(disc)
    full = _replay(pat, dtn, list(range(len(disc.leaves))))
    order = [7, 2, 11, 0, 5, 9, 1, 3, 10, 4, 8, 6]
    acc = [np.zeros(pat.nnz[0]), np.zeros(pat.nnz[1])]
    for chunk in (order[:5], order[5:]):
        part = _replay(pat, dtn[chunk], chunk)
        acc[0] += part[0]
        acc[1] += part[1]
    assert np.array_equal(acc[0], full[0]) and np.array_equal(acc[1], full[1])


def test_resident_job_table_matches_per_flush_jobs():
    pat = InterfacePattern(_disc((3, 2, 2), 5, "drop"))
    n = len(pat.leaf_jobs)
    per_flush = pat.jobs_for(range(n))
    assert np.array_equal(pat.all_jobs, per_flush)  # position == global id for the full range
    lo, hi = pat.job_offsets[4], pat.job_offsets[9]
    sub = pat.jobs_for(range(4, 9))
    assert np.array_equal(pat.all_jobs[lo:hi, 1:], sub[:, 1:])
    assert np.array_equal(pat.all_jobs[lo:hi, 0] - 4, sub[:, 0])


def test_every_entry_has_at_most_two_contributors():
    """The bit-exactness argument: 0 + x + y is order independent."""
    disc = _disc((3, 2, 2), 5, "drop")
    pat = InterfacePattern(disc)
    m = len(disc.leaves[0].boundary_ids)
    count = _replay(pat, np.ones((len(disc.leaves), m, m)), list(range(len(disc.leaves))))
    assert count[0].max() == 2 and count[0].min() >= 1
    assert count[1].max() == 1


@pytest.mark.gpu
@pytest.mark.parametrize("boxes,p,mode", CASES)
def test_device_scatter_is_bit_exact(boxes, p, mode):
    import torch
    from paper_2503_04033_b200.assembly import DeviceAssembler
    disc = _disc(boxes, p, mode)
    m = len(disc.leaves[0].boundary_ids)
    dtn = np.random.default_rng(7).standard_normal((len(disc.leaves), m, m))
    t_ref, c_ref = _host(disc, dtn)
    asm = DeviceAssembler(InterfacePattern(disc), 0)
    ids = list(range(len(disc.leaves)))
    perm = list(np.random.default_rng(1).permutation(len(ids)))
    flushes = [ids[lo:lo + 5] for lo in range(0, len(ids), 5)]  # contiguous: resident job table
    flushes = flushes[1::2]
    done = {i for f in flushes for i in f}
    rest = [int(i) for i in perm if i not in done]  # non-contiguous: per-flush job tables
    flushes += [rest[:len(rest) // 2], rest[len(rest) // 2:]]
    for chunk in flushes:
        if chunk:
            asm.add(torch.from_numpy(dtn[chunk]).cuda(), chunk)
    t, c = asm.finish()
    _same(t, t_ref)
    _same(c, c_ref)


@pytest.mark.gpu
@pytest.mark.parametrize("boxes,p", [((2, 2, 2), 8), ((4, 3), 10)])
def test_build_device_and_host_assembly_identical(boxes, p, monkeypatch):
    from paper_2503_04033_b200.condensation import build
    from paper_2503_04033_b200.local_ops import isotropic_field
    disc = _disc(boxes, p, "drop")
    field = isotropic_field(len(boxes), zeroth=lambda x: -150.0 * (1.0 - 0.5 * np.exp(-((x - 0.4) ** 2).sum(1) / 0.05)))
    monkeypatch.setenv("HPS_HOST_ASSEMBLY", "1")
    host = build(disc, field)
    monkeypatch.setenv("HPS_HOST_ASSEMBLY", "0")
    dev = build(disc, field)
    _same(dev.t, host.t)
    _same(dev.dirichlet_coupling, host.dirichlet_coupling)


@pytest.mark.gpu
def test_build_flushes_and_workspace_release():
    """A budget of a few staged maps (many flushes, partial waves) gives the same T and
    C bit for bit as one flush; the staged bytes stay within memory_budget; the leaf
    engine's workspace is reported, can be released and is re-allocated on demand."""
    from paper_2503_04033_b200 import BatchSchedule, make_problem
    from paper_2503_04033_b200.condensation import build
    spec = make_problem("bump_helmholtz", d=3, kappa=20.0)
    disc = build_discretization(spec.domain, MeshConfig((3, 2, 2), 8))
    one = build(disc, spec.coeffs, BatchSchedule())
    small = build(disc, spec.coeffs, BatchSchedule(resident_limit=5))   # 12 leaves in 3 flushes
    assert small.peak_workspace_bytes < one.peak_workspace_bytes <= BatchSchedule().memory_budget
    _same(small.t, one.t)
    _same(small.dirichlet_coupling, one.dirichlet_coupling)
    eng = small.engine
    held, slots = eng.workspace()
    assert held > 0 and slots >= 1 and small.device_workspace_bytes > 0
    eng.release()
    assert eng.workspace() == (0, 0)
    again = build(disc, spec.coeffs, BatchSchedule(resident_limit=5))
    _same(again.t, one.t)


@pytest.mark.parametrize("boxes,p,mode", CASES)
def test_vector_jobs_reproduce_host_flux_sum(boxes, p, mode):
    """g_b = -(sum of interface fluxes) through the vector jobs == the host loop
    g_b[t_rows] -= flux (reference condensation.py:314-323), bit for bit."""
    disc = _disc(boxes, p, mode)
    m = len(disc.leaves[0].boundary_ids)
    flux = np.random.default_rng(5).standard_normal((len(disc.leaves), m))
    tpl = LeafTemplate(disc.leaf_widths, disc.p, disc.corner_mode, False)
    dof_map = _make_dof_map(disc, tpl)
    ref = np.zeros(disc.n_interface)
    for k, dofs in enumerate(dof_map.per_leaf):
        ref[dofs.t_rows] -= flux[k][dofs.interface_mask]
    pat = InterfacePattern(disc)
    acc = np.zeros(disc.n_interface)
    for k, r0, c0, nr, nc, tgt, base, stride in pat.jobs_for(range(len(disc.leaves)), vectors=True):
        assert (c0, nc, tgt, stride) == (0, 1, 0, 1)
        np.add.at(acc, base + np.arange(nr), flux[k, r0:r0 + nr])
    assert np.array_equal(-acc, ref)


@pytest.mark.gpu
def test_reduce_load_device_and_host_identical(monkeypatch):
    from paper_2503_04033_b200 import make_problem
    from paper_2503_04033_b200.condensation import build, reduce_load
    spec = make_problem("bump_helmholtz", d=3, kappa=20.0)
    disc = build_discretization(spec.domain, MeshConfig((3, 2, 2), 8))
    sys_ = build(disc, spec.coeffs)
    assert sys_.pattern is not None
    v_dev, g_dev = reduce_load(disc, spec.coeffs, spec.f, spec.g, sys_)
    monkeypatch.setenv("HPS_HOST_ASSEMBLY", "1")
    v_host, g_host = reduce_load(disc, spec.coeffs, spec.f, spec.g, sys_)
    assert np.array_equal(g_dev, g_host)
    assert all(np.array_equal(a, b) for a, b in zip(v_dev, v_host))


def test_cached_pattern_indices_are_read_only():
    """T and C share the cached pattern's index arrays: an in-place structural edit
    of a returned matrix raises instead of corrupting later builds (advisor finding)."""
    disc = _disc((2, 2, 1), 6, "drop")
    pat = InterfacePattern(disc)
    t, c = pat.matrices(np.ones(pat.nnz[0]), np.ones(pat.nnz[1]))
    before = pat.indptr[0].copy()
    with pytest.raises(ValueError):
        t.eliminate_zeros()
    assert np.array_equal(pat.indptr[0], before)
    t2 = t.copy()            # a copy is the user's own
    t2.data[:] = 0.0
    t2.eliminate_zeros()
    assert t2.nnz == 0 and t.nnz == pat.nnz[0]


def test_pattern_is_built_once_per_discretization():
    from paper_2503_04033_b200.assembly import pattern_for
    disc = _disc((2, 2, 1), 6, "drop")
    assert pattern_for(disc) is pattern_for(disc)
    assert pattern_for(_disc((2, 2, 1), 6, "drop")) is not pattern_for(disc)
