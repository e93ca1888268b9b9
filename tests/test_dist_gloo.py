"""Multi-process (gloo, CPU) coverage of the multi-rank solver stages.

``build``, ``reduce_load`` and ``solve`` split the leaves by index over the
ranks of an initialized torch.distributed group (reference worker pool,
condensation.py:248-264, 325-333, 385-391).  Here every rank's GPU is stood in
for by the CPU oracle (tests/hps_fakes.py); the sharding, flushes and collectives
run unchanged over gloo.  The bar is bit-exact against one process: the same T,
C, g_b and solution.
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
    spec = make_problem("helmholtz_green", d=3, kappa=6.0)
    return spec, build_discretization(spec.domain, MeshConfig((3, 2, 2), 6))


def _schedule(**kw):
    from paper_2503_04033_b200.condensation import BatchSchedule
    # a small budget: several flushes per rank (5 staged blocks of 8 * 96^2 bytes per flush)
    return BatchSchedule(memory_budget=5 * 8 * 96 ** 2 + 4 * 96 ** 2, **kw)


def _run(distributed):
    from paper_2503_04033_b200.condensation import build, reduce_load, solve
    spec, disc = _problem()
    sys_ = build(disc, spec.coeffs, _schedule(distributed=distributed))
    v_list, g_b = reduce_load(disc, spec.coeffs, spec.f, spec.g, sys_)
    report = solve(sys_, v_list, g_b, spec.g)
    return sys_, v_list, g_b, report


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import hps_fakes as _fakes
        engines = _fakes.install()
        sys_, v_list, g_b, report = _run(None)
        shard = sys_.shard
        assert shard is not None and shard.world == world and shard.rank == rank
        own = set(shard.ids)
        assert all((v is not None) == (i in own) for i, v in enumerate(v_list))
        assert sys_.peak_workspace_bytes <= sys_.schedule.memory_budget
        launches = sum(e.launches for e in engines)
        res = dict(u=report.u, residual=report.residual, launches=launches,
                   start=shard.start, stop=shard.stop)
        if rank == 0:
            res.update(t_data=sys_.t.data, t_indices=sys_.t.indices, t_indptr=sys_.t.indptr,
                       c_data=sys_.dirichlet_coupling.data, g_b=g_b)
        else:
            assert sys_.t is None and sys_.factorization is None and g_b is None
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_multi_rank_build_load_solve_match_single_process(tmp_path, world, monkeypatch):
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn")
    import hps_fakes as _fakes
    from paper_2503_04033_b200 import condensation
    monkeypatch.setattr(condensation, "_engine_for", condensation._engine_for)
    monkeypatch.setattr(condensation, "DeviceAssembler", condensation.DeviceAssembler)
    _fakes.install()
    sys_, v_list, g_b, report = _run(False)
    assert sys_.shard is None
    r0 = np.load(tmp_path / "rank0.npz")
    # T, C and g_b summed onto the root: bit-identical to one process
    assert np.array_equal(r0["t_indptr"], sys_.t.indptr)
    assert np.array_equal(r0["t_indices"], sys_.t.indices)
    assert np.array_equal(r0["t_data"], sys_.t.data)
    assert np.array_equal(r0["c_data"], sys_.dirichlet_coupling.data)
    assert np.array_equal(r0["g_b"], g_b)
    spans = []
    for r in range(world):
        res = np.load(tmp_path / f"rank{r}.npz")
        # every rank returns the same assembled solution and residual
        assert np.array_equal(res["u"], report.u)
        assert float(res["residual"]) == report.residual
        spans.append((int(res["start"]), int(res["stop"])))
        assert int(res["launches"]) >= 1
    assert spans == [shard_range(len(sys_.disc.leaves), world, r) for r in range(world)]
    # and the solution is the manufactured one to the accuracy of p = 6 leaves
    spec, disc = _problem()
    exact = spec.exact(disc.nodes)
    assert np.linalg.norm(report.u - exact) / np.linalg.norm(exact) < 2e-3


def test_flush_respects_budgets():
    """Flushes of two device waves (2 x slots leaves), bounded by resident_limit and
    by memory_budget for the host staging (the reference's peak_workspace_bytes <=
    budget contract, condensation.py:255-263, 291); the results do not depend on it."""
    import hps_fakes as _fakes
    from paper_2503_04033_b200 import condensation
    saved = condensation._engine_for, condensation.DeviceAssembler
    try:
        engines = _fakes.install(slots=3)
        spec, disc = _problem()
        sched = _schedule(distributed=False)
        sys_ = condensation.build(disc, spec.coeffs, sched)
        pack_bytes = 8 * 4 * 64                   # ncoef x n doubles per leaf
        assert sys_.peak_workspace_bytes == 2 * 6 * pack_bytes <= sched.memory_budget
        assert engines[-1].launches == 2          # 12 leaves, flushes of 2 x 3 slots
        # (the reference's resolve() caps resident_limit by the budget: at most 3 maps here)
        sys2 = condensation.build(disc, spec.coeffs, _schedule(distributed=False, resident_limit=3))
        assert engines[-1].launches == 4 and sys2.peak_workspace_bytes == 2 * 3 * pack_bytes
        assert np.array_equal(sys2.t.data, sys_.t.data)
        # a budget that holds the staging of only two leaves' packs bounds the flush to one leaf
        tight = condensation.BatchSchedule(memory_budget=2 * pack_bytes + 8 * 64 ** 2 * 4, distributed=False)
        with pytest.raises(condensation.ConfigError):
            tight.resolve(disc.p, disc.d, disc.corner_mode)   # cannot hold one leaf workspace
        res = _schedule().resolve(disc.p, disc.d, disc.corner_mode)
        eng = engines[-1]
        assert condensation._flush_size(res, eng, 12, device_staging=False) == 5  # 5.5 maps in budget
        res.memory_budget = 3 * pack_bytes
        assert condensation._flush_size(res, eng, 12, device_staging=True) == 1
    finally:
        condensation._engine_for, condensation.DeviceAssembler = saved


def test_max_over_ranks_single_process():
    from paper_2503_04033_b200.sharding import max_over_ranks
    assert max_over_ranks(3.5) == 3.5


def test_bench_leaf_shards_cover_the_grid():
    """bench.py --gpus N: rank r owns leaves [L r / N, L (r + 1) / N) of ONE grid;
    the configs[3] share of rank r is the r-th eighth."""
    import bench
    for world in (1, 2, 4, 8):
        ids = [bench.shard_ids(4096, world, r) for r in range(world)]
        assert sum(ids, []) == list(range(4096))
    assert bench.shard_ids(4096, 8, 0) == list(range(512))
    assert bench.shard_ids(4096, 8, 3)[0] == 1536
