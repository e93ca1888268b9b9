"""bench.py's reference arm under torchrun (CPU only): rank 0 alone runs the CPU
reference and prints one JSON line; the other ranks exit 0 without work."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(cmd, env_extra=None):
    env = dict(os.environ, OMP_NUM_THREADS="2", OPENBLAS_NUM_THREADS="2", HPS_REF_WORKERS="2",
               MASTER_ADDR="127.0.0.1")
    env.update(env_extra or {})
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)


def _lines(stdout):
    return [json.loads(s) for s in stdout.splitlines() if s.startswith("{")]


def test_reference_arm_single_process():
    res = _run([sys.executable, "bench.py", "--impl", "reference", "--p", "8", "--boxes", "2",
                "--steps", "1", "--warmup", "1", "--ref-seconds", "2"])
    assert res.returncode == 0, res.stderr[-2000:]
    (line,) = _lines(res.stdout)
    assert line["impl"] == "reference" and line["n_gpus"] == 1
    assert line["metric"] == "leaf DtN maps/sec" and line["value"] > 0
    assert line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    # the installed reference (baseline/_ref) when present, else the oracle port
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["cpu_baseline"]["cores"] == 2  # HPS_REF_WORKERS
    assert line["config"]["p"] == 8 and line["config"]["leaves_per_gpu"] == 8
    # what ran is what the line says: steps x ms_per_step is the measured time
    assert line["leaves_timed"] == line["steps"] * line["config"]["sample_leaves"]
    assert abs(line["value"] * line["steps"] * line["ms_per_step"] / 1e3 - line["leaves_timed"]) \
        <= 1e-6 * line["leaves_timed"]


def test_reference_arm_under_torchrun_prints_one_line():
    res = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                "--master-addr", "127.0.0.1", "--master-port", "29561", "bench.py", "--impl",
                "reference", "--gpus", "2", "--p", "8", "--boxes", "2", "--steps", "1",
                "--warmup", "1", "--ref-seconds", "2"])
    assert res.returncode == 0, res.stderr[-2000:]
    (line,) = _lines(res.stdout)
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["leaves_per_gpu"] == 4   # the 2x2x2 grid split by leaf index


def test_bench_parity_spot_check_spreads_over_the_grid():
    """bench.py's parity leaves: 8 per rank, the bump-centre leaf and the fixture
    leaves first, the rest spread over the share."""
    import bench
    ids = list(range(4096))
    chosen = bench.spread_sample(ids, 8, must=[bench.centre_leaf(16), 375])
    assert chosen[:2] == [1911, 375] and len(set(chosen)) == 8
    assert max(chosen) - min(chosen) > 3000
