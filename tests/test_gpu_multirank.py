"""Multi-rank solver stages and the bench's N-rank line through the REAL engine.

test_dist_gloo.py covers the sharding / flush / collective logic with the CPU
oracle standing in for each rank's GPU.  Here two ranks run the CUDA engine
(libhps_leaf.so) for their own leaf shards, on the one GPU of the test box,
with the exchanges over gloo (CPU copies; NCCL refuses two ranks on one
device).  The ranks' kernels never wait on each other — the only coupling is
the host-side reduce / broadcast / gather of build, reduce_load and solve
(reference worker pool, condensation.py:248-264, 325-333, 385-391) — so this
checks the multi-rank path bit for bit against one process; it says nothing
about multi-GPU speed.
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    from paper_2503_04033_b200.geometry import MeshConfig, build_discretization
    from paper_2503_04033_b200.problems import make_problem
    spec = make_problem("helmholtz_green", d=3, kappa=6.0)
    return spec, build_discretization(spec.domain, MeshConfig((3, 2, 2), 8))


def _run(distributed):
    from paper_2503_04033_b200.condensation import BatchSchedule, build, reduce_load, solve
    spec, disc = _problem()
    # two leaves per flush: several flushes (launches) per rank
    sched = BatchSchedule(memory_budget=4 << 20, resident_limit=2, distributed=distributed)
    sys_ = build(disc, spec.coeffs, sched)
    v_list, g_b = reduce_load(disc, spec.coeffs, spec.f, spec.g, sys_)
    report = solve(sys_, v_list, g_b, spec.g)
    return sys_, v_list, g_b, report


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys_, v_list, g_b, report = _run(None)
        shard = sys_.shard
        assert shard is not None and shard.world == world and shard.rank == rank
        res = dict(u=report.u, residual=report.residual, start=shard.start, stop=shard.stop)
        if rank == 0:
            res.update(t_data=sys_.t.data, t_indices=sys_.t.indices, t_indptr=sys_.t.indptr,
                       c_data=sys_.dirichlet_coupling.data, g_b=g_b)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_the_cuda_engine_match_one_process(tmp_path):
    from paper_2503_04033_b200.sharding import shard_range
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn")
    sys_, v_list, g_b, report = _run(False)
    assert sys_.shard is None
    r0 = np.load(tmp_path / "rank0.npz")
    assert np.array_equal(r0["t_indptr"], sys_.t.indptr)
    assert np.array_equal(r0["t_indices"], sys_.t.indices)
    assert np.array_equal(r0["t_data"], sys_.t.data)
    assert np.array_equal(r0["c_data"], sys_.dirichlet_coupling.data)
    assert np.array_equal(r0["g_b"], g_b)
    spans = []
    for r in range(world):
        res = np.load(tmp_path / f"rank{r}.npz")
        assert np.array_equal(res["u"], report.u)
        assert float(res["residual"]) == report.residual
        spans.append((int(res["start"]), int(res["stop"])))
    assert spans == [shard_range(len(sys_.disc.leaves), world, r) for r in range(world)]
    spec, disc = _problem()
    exact = spec.exact(disc.nodes)
    assert np.linalg.norm(report.u - exact) / np.linalg.norm(exact) < 2e-3


def test_bench_two_rank_line_plumbing():
    """bench.py launched as the driver launches N = 2 (torchrun), with gloo so both
    ranks fit on one GPU: one JSON line, the grid split by leaf index, max over ranks,
    parity on every rank.  (Timing of ranks sharing one GPU is not a scaling number.)"""
    env = dict(os.environ, HPS_BENCH_BACKEND="gloo")
    res = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                          str(_free_port()), "bench.py", "--gpus", "2", "--p", "8", "--boxes", "4",
                          "--steps", "3", "--warmup", "3", "--no-cpu", "--e2e-steps", "1",
                          "--configs3-steps", "0"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [json.loads(x) for x in res.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["n_gpus"] == 2 and line["config"]["leaves_per_gpu"] == 32
    assert line["parity"]["ok"] and line["parity"]["all_ranks_ok"]
    assert line["e2e"]["leaves_per_gpu"] == 32
    assert abs(line["value"] * line["ms_per_step"] / 1e3 - 64) <= 1e-6 * 64
