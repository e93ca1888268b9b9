"""Multi-process (world_size 2, gloo, CPU) coverage of the leaf-sharded build path.

Each rank reduces its contiguous leaf shard (here with the CPU oracle standing in
for the rank's GPU) and the blocks are gathered to rank 0 in leaf order; the
result must equal the single-process computation.  Also checks the
max-over-ranks timing rule.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2503_04033_b200.sharding import shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 64, 4097):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _problem():
    from paper_2503_04033_b200.geometry import MeshConfig, build_discretization
    from paper_2503_04033_b200.problems import make_problem
    spec = make_problem("bump_helmholtz", d=3, kappa=12.0)
    return spec, build_discretization(spec.domain, MeshConfig((3, 2, 2), 6))


def _oracle_compute(disc):
    from oracle import hps_oracle as O
    tpl = O.OracleTemplate(disc.leaf_widths, disc.p)

    def compute(pack):
        return np.stack([O.leaf_dtn(tpl, c[:3].T, None, c[3])[0] for c in pack])
    return compute


def _worker(rank, world, port, out_path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_04033_b200.sharding import max_over_ranks, sharded_dtn
        spec, disc = _problem()
        blocks = sharded_dtn(disc, spec.coeffs, world, rank, compute=_oracle_compute(disc))
        slowest = max_over_ranks(float(rank + 1))
        if rank == 0:
            np.savez(out_path, blocks=blocks, slowest=slowest)
        else:
            assert blocks is None
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_build_matches_single_process(tmp_path):
    out = str(tmp_path / "dist.npz")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, start_method="spawn")
    res = np.load(out)
    spec, disc = _problem()
    from paper_2503_04033_b200.local_ops import pack_coefficients
    from paper_2503_04033_b200.condensation import interior_points
    full = _oracle_compute(disc)(pack_coefficients(spec.coeffs,
                                                   interior_points(disc, range(len(disc.leaves))),
                                                   len(disc.leaves)))
    assert np.array_equal(res["blocks"], full)
    assert float(res["slowest"]) == 2.0


def _replay_scatter(pattern, dtn, ids):
    """numpy replay of hps_interface_scatter (the rank's GPU in this CPU test)."""
    out = [np.zeros(pattern.nnz[0]), np.zeros(pattern.nnz[1])]
    for k, r0, c0, nr, nc, tgt, base, stride in pattern.jobs_for(ids):
        idx = base + np.arange(nr)[:, None] * stride + np.arange(nc)[None, :]
        np.add.at(out[tgt], idx, dtn[k, r0:r0 + nr, c0:c0 + nc])
    return out


def _interface_worker(rank, world, port, out_path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_04033_b200.sharding import sharded_interface
        spec, disc = _problem()
        res = sharded_interface(disc, spec.coeffs, world, rank, compute=_oracle_compute(disc),
                                scatter=_replay_scatter)
        if rank == 0:
            t, c = res
            np.savez(out_path, t_data=t.data, t_indices=t.indices, t_indptr=t.indptr,
                     c_data=c.data, c_indices=c.indices, c_indptr=c.indptr)
        else:
            assert res is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_interface_reduce_matches_host_assembly(tmp_path, world):
    """Partial CSR values of T and C per rank, one sum-reduce: bit-identical to
    the single-process host scatter of all DtN maps."""
    out = str(tmp_path / "iface.npz")
    mp.start_processes(_interface_worker, args=(world, _free_port(), out), nprocs=world,
                       start_method="spawn")
    res = np.load(out)
    spec, disc = _problem()
    from paper_2503_04033_b200.condensation import (_make_dof_map, finalize_host, interior_points,
                                                    scatter_leaf_blocks)
    from paper_2503_04033_b200.local_ops import LeafTemplate, pack_coefficients
    from paper_2503_04033_b200.sparse_backend import SparseMatrix
    ids = list(range(len(disc.leaves)))
    full = _oracle_compute(disc)(pack_coefficients(spec.coeffs, interior_points(disc, ids), len(ids)))
    dof_map = _make_dof_map(disc, LeafTemplate(disc.leaf_widths, disc.p, disc.corner_mode, False))
    tb, cr, cc, cv = SparseMatrix(disc.n_interface), [], [], []
    scatter_leaf_blocks(dof_map, ids, full, tb, cr, cc, cv)
    t, c = finalize_host(tb, cr, cc, cv, disc.n_interface, disc.n_dirichlet)
    for name, ref in (("t", t), ("c", c)):
        assert np.array_equal(res[f"{name}_indptr"], ref.indptr)
        assert np.array_equal(res[f"{name}_indices"], ref.indices)
        assert np.array_equal(res[f"{name}_data"], ref.data)
