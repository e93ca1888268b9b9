"""Leaf DtN throughput on B200: the two-level HPS solver's batched leaf-box reduction.

Headline workload (BASELINE.json configs[2]): 3D variable-coefficient Helmholtz
    -Lap u - kappa^2 b(x) u,  b(x) = 1 - 0.5 exp(-|x - c|^2 / (2 * 0.15^2)),
p = 16 Chebyshev nodes per axis, one 16 x 16 x 16 leaf grid on the unit cube,
kappa = 40.  One step = the DtN maps of every leaf of the rank's share
(operator assembly, pivoted LU of A_ii, Schur complement), inputs resident in
HBM.  Under torchrun the grid is split by leaf index — rank r owns leaves
[L r / N, L (r + 1) / N) — with no collective on the data path (strong
scaling: the grid is the same at every N).

Second workload, reported as the ``configs3`` sub-object (BASELINE configs[3]):
p = 20, 16^3 leaves, kappa = 80, sharded across 8 GPUs by leaf index; rank r
times share r (leaves 512 r .. 512 r + 511), so at N = 1 it is rank 0's share.

Prints ONE JSON line (rank 0).  ``--impl reference`` times the reference's own
CPU path on the host cores instead: ``steklov.local_ops.build_leaf_factors``
from the installed reference (``baseline/_ref``) over the reference's worker
pool, or — if that install is missing — the oracle port in ``oracle/``.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAK_FP64_TFLOPS = 37.1   # measured DMMA issue peak, profiles/r01_fp64_probe_dmma_dfma.log
PEAK_FP64_CUBLAS = 35.5   # measured cuBLAS DGEMM, profiles/r01_fp64_probe_cublas_cusolver.log
TOL = 1e-10               # north star: relative Frobenius error vs the CPU reference
CONFIGS3 = {"p": 20, "boxes": 16, "kappa": 80.0, "shards": 8}
FIXTURES = os.path.join(ROOT, "tests", "golden", "bench_cases.npz")
METRIC = "leaf DtN maps/sec"
UNIT = "leaf DtN maps/s"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--p", type=int, default=16)
    ap.add_argument("--boxes", type=int, default=16, help="leaf boxes per axis of the grid")
    ap.add_argument("--kappa", type=float, default=40.0)
    ap.add_argument("--field", default="bump", choices=["bump", "const"],
                    help="bump: variable-coefficient b(x) (configs 2-3); const: b = 1 (configs[1])")
    ap.add_argument("--leaves", type=int, default=0, help="override leaves per rank (profiling)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=60.0,
                    help="reference arm: CPU seconds over the timed steps")
    ap.add_argument("--configs3-steps", type=int, default=5,
                    help="timed steps of the p = 20 configs[3] share (0: skip)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args(argv)


# Plumbing check only (tests/test_gpu_multirank.py): HPS_BENCH_BACKEND=gloo runs the
# N-rank line on fewer GPUs (rank r on GPU r mod count, host collectives).  The
# ranks' kernels never wait on each other, but ranks sharing a GPU share its SMs,
# so such a line checks the sharding / barrier / max-over-ranks plumbing, not speed.
BACKEND = os.environ.get("HPS_BENCH_BACKEND", "nccl")


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if BACKEND == "gloo" and world > 1:
        import torch
        local %= max(torch.cuda.device_count(), 1)
    return world, rank, local


def bump_b(x):
    r2 = ((x - 0.5) ** 2).sum(axis=1)
    return 1.0 - 0.5 * np.exp(-r2 / (2 * 0.15 ** 2))


def host_mem_available():
    """MemAvailable of the node in bytes (Linux), or a large number if unknown."""
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 1 << 50


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def pinned_host(shape):
    """Page-locked float64 host array of exactly this size (cudaHostRegister on a numpy
    buffer; the torch pinned allocator rounds large requests up to a power of two)."""
    import torch
    a = np.empty(shape, dtype=np.float64)
    torch.cuda.check_error(torch.cuda.cudart().cudaHostRegister(a.ctypes.data, a.nbytes, 0))
    return a


def unpin_host(a):
    import torch
    torch.cuda.check_error(torch.cuda.cudart().cudaHostUnregister(a.ctypes.data))


def shard_ids(n_leaves, world, rank):
    from paper_2503_04033_b200.sharding import shard_range
    start, stop = shard_range(n_leaves, world, rank)
    return list(range(start, stop))


def make_shard(p, boxes, kappa, rank=0, world=1, leaves_override=0, field="bump", leaf_ids=None):
    """Coefficient packs (L, 4, n) of leaves of the boxes^3 grid on the unit cube.

    ``leaf_ids`` (flat C-order indices of the grid) default to rank's leaf-index
    share of the grid; ``leaves_override`` takes the first L leaves (cycling),
    for profiling tools.  field "bump": -Lap u - kappa^2 b(x) u (configs 2-3);
    "const": b = 1 (configs[1]).  The nodes are the reference's leaf grid
    (local_ops.py build_leaf_operator: lo + h * ref_offsets)."""
    from paper_2503_04033_b200.local_ops import LeafTemplate
    h = 1.0 / boxes
    tpl = LeafTemplate((h, h, h), p, "drop", False)
    if leaf_ids is None:
        leaf_ids = ([k % boxes ** 3 for k in range(leaves_override)] if leaves_override
                    else shard_ids(boxes ** 3, world, rank))
    leaf_ids = np.asarray(leaf_ids, dtype=np.int64)
    L = len(leaf_ids)
    n = tpl.n_interior
    inner = tpl.ref_offsets[1:-1]
    q = len(inner)
    pack = np.empty((L, 4, n))
    pack[:, :3, :] = 1.0
    idx = np.stack(np.unravel_index(leaf_ids, (boxes,) * 3), axis=1).astype(float)
    for k0 in range(0, L, 256):
        lo = idx[k0:k0 + 256] * h
        B = len(lo)
        g = [lo[:, a, None] + h * inner[None, :] for a in range(3)]
        X = np.broadcast_to(g[0][:, :, None, None], (B, q, q, q))
        Y = np.broadcast_to(g[1][:, None, :, None], (B, q, q, q))
        Z = np.broadcast_to(g[2][:, None, None, :], (B, q, q, q))
        pts = np.stack([X, Y, Z], axis=-1).reshape(-1, 3)
        b = bump_b(pts) if field == "bump" else np.ones(len(pts))
        pack[k0:k0 + B, 3, :] = (-kappa * kappa * b).reshape(B, n)
    return tpl, pack


def centre_leaf(boxes):
    """Flat index of the leaf whose upper corner is the bump centre (0.5, 0.5, 0.5)."""
    c = max(boxes // 2 - 1, 0)
    return int(np.ravel_multi_index((c, c, c), (boxes,) * 3))


def spread_sample(ids, k, must=()):
    """k leaf ids of ``ids``: the ``must`` ids that are present, then evenly spaced ones."""
    ids = list(ids)
    present = set(ids)
    out = [i for i in dict.fromkeys(must) if i in present][:k]
    rest = [i for i in ids if i not in set(out)]
    need = min(k - len(out), len(rest))
    if need > 0:
        out += [rest[j] for j in np.linspace(0, len(rest) - 1, num=need).round().astype(int)]
    return out


def low_discrepancy_ids(n_leaves, first):
    """Every leaf id once, ``first`` leading, then a golden-ratio sequence over the grid
    (each prefix spreads over the whole grid)."""
    phi = (np.sqrt(5.0) - 1.0) / 2.0
    seq = np.floor(((np.arange(4 * n_leaves) * phi) % 1.0) * n_leaves).astype(int)
    out, seen = [first], {first}
    for i in seq.tolist() + list(range(n_leaves)):
        if i not in seen:
            seen.add(i)
            out.append(i)
    return out


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) == 7:
                    rows.append(parts)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        pw = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = [nm for i, nm in enumerate(names) if any(r[3 + i] == "Active" for r in rows)]
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(pw) if pw else None,
                "power_w_median": float(np.median(pw)) if pw else None}


def traffic_per_leaf(p):
    """DRAM bytes per leaf from the committed ncu --set full capture at this order."""
    for name in (f"r02c_final6_ncu_summary_p{p}.json", f"r02c_final5_ncu_summary_p{p}.json", f"r02c_final4_ncu_summary_p{p}.json", f"r02c_final2_ncu_summary_p{p}.json", f"r02c_final_ncu_summary_p{p}.json", f"r02c_ncu_summary_p{p}.json", f"r02b_ncu_summary_p{p}.json",
                 f"r02_ncu_summary_p{p}.json",
                 "r01_ncu_summary.json"):
        path = os.path.join(ROOT, "profiles", name)
        try:
            s = json.load(open(path))
        except (OSError, ValueError):
            continue
        if int(s.get("p", 16)) == p and "traffic_bytes_per_leaf" in s:
            return s["traffic_bytes_per_leaf"], "profiles/" + name
    return None, None


# ---------------------------------------------------------------------------
# the reference's CPU path (reference arm and cpu_baseline)
# ---------------------------------------------------------------------------

class ReferenceCPU:
    """Per-leaf DtN maps on the host cores, through the reference's own API when it is
    installed (baseline/_ref: steklov.local_ops.build_leaf_factors on the leaf grid the
    reference's build() uses, condensation.py:218-221, over a worker pool like its
    ``BatchSchedule.workers``; one BLAS thread per worker), else the oracle port
    (oracle/hps_oracle.py, the same algorithm restated)."""

    def __init__(self, p, boxes, kappa, field, workers=0):
        self.p, self.boxes, self.kappa, self.field = p, boxes, kappa, field
        self.workers = workers or int(os.environ.get("HPS_REF_WORKERS", "0")) or host_cores()
        self.h = 1.0 / boxes
        ref = os.path.join(ROOT, "baseline", "_ref")
        self.kind = "port"
        try:
            if os.path.isdir(os.path.join(ref, "steklov")):
                if ref not in sys.path:
                    sys.path.insert(0, ref)
                from steklov import local_ops as SL
                self.SL = SL
                self.kind = "reference"
        except Exception:
            self.kind = "port"
        if self.kind == "reference":
            SL = self.SL
            if field == "bump":
                zeroth = lambda x: -kappa * kappa * bump_b(x)  # noqa: E731
            else:
                zeroth = lambda x: np.full(x.shape[0], -kappa * kappa)  # noqa: E731
            self.coeffs = SL.isotropic_field(3, zeroth=zeroth)
            self.tpl = SL.LeafTemplate(np.array([self.h] * 3), p, SL.DROP_CORNERS, False)
        else:
            from oracle import hps_oracle as O
            self.O = O
            self.otpl = O.OracleTemplate((self.h,) * 3, p)

    def leaf(self, leaf_id):
        if self.kind == "reference":
            lo = np.asarray(np.unravel_index(leaf_id, (self.boxes,) * 3), dtype=float) * self.h
            nodes = []
            for k in range(3):
                x = lo[k] + self.h * self.tpl.ref_offsets
                x[0], x[-1] = lo[k], lo[k] + self.h
                nodes.append(x)
            grid = self.tpl.leaf_grid(nodes)
            return self.SL.build_leaf_factors(self.tpl, self.coeffs, grid).dtn
        _, pack = make_shard(self.p, self.boxes, self.kappa, field=self.field, leaf_ids=[leaf_id])
        return self.O.leaf_dtn(self.otpl, pack[0, :3].T, None, pack[0, 3])[0]

    def run(self, ids):
        """DtN maps of ``ids`` over the worker pool; returns seconds."""
        from concurrent.futures import ThreadPoolExecutor
        from threadpoolctl import threadpool_limits
        t0 = time.perf_counter()
        with threadpool_limits(limits=1, user_api="blas"):
            with ThreadPoolExecutor(max_workers=self.workers) as pool:
                list(pool.map(self.leaf, ids))
        return time.perf_counter() - t0

    def describe(self):
        if self.kind == "reference":
            return (f"reference steklov.local_ops.build_leaf_factors (baseline/_ref, scipy LAPACK "
                    f"getrf/getrs + numpy GEMM) on {self.workers} worker threads x 1 BLAS thread")
        return (f"oracle port of build_leaf_factors (numpy/scipy LAPACK getrf/getrs + GEMM) on "
                f"{self.workers} worker threads x 1 BLAS thread")


def cpu_baseline(p, boxes, kappa, field, seconds):
    """Bounded CPU sample of the workload (rank 0, N = 1 leg of the GPU line)."""
    ref = ReferenceCPU(p, boxes, kappa, field)
    order = low_discrepancy_ids(boxes ** 3, centre_leaf(boxes))
    done, spent = 0, 0.0
    while spent < seconds or done == 0:
        ids = order[done:done + ref.workers]
        spent += ref.run(ids)
        done += len(ids)
    return {"value": done / spent, "unit": UNIT, "cores": ref.workers, "kind": ref.kind,
            "sample": f"{done} leaves spread over the {boxes}^3 grid (bump-centre leaf first), "
                      f"{ref.describe()}, {spent:.1f} s"}


def config_of(args, world, leaves_per_gpu):
    p, boxes = args.p, args.boxes
    n, m = (p - 2) ** 3, 6 * (p - 2) ** 2
    kind = ("3D variable-coefficient Helmholtz b(x) (Gaussian bump)" if args.field == "bump"
            else "3D constant-coefficient Helmholtz")
    share = (f"{boxes}x{boxes}x{boxes} leaves" if not args.leaves else
             f"{leaves_per_gpu} leaves per GPU of a {boxes}x{boxes}x{boxes} grid (profiling override)")
    return {"workload": f"{kind}, p={p}, {share}, kappa={args.kappa:g}", "p": p,
            "grid": [boxes] * 3, "leaves": (args.leaves * world) if args.leaves else boxes ** 3,
            "leaves_per_gpu": leaves_per_gpu, "n_interior": n, "n_boundary": m,
            "kappa": args.kappa, "field": args.field,
            "l2": "inputs (coefficients %.0f MB) and outputs (%.1f GB) per GPU exceed the 126 MB L2"
                  % (leaves_per_gpu * 4 * n * 8 / 1e6, leaves_per_gpu * m * m * 8 / 1e9),
            "parallelism": f"leaf-index shards x{world}, no data-path collective"}


def reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    ref = ReferenceCPU(args.p, args.boxes, args.kappa, args.field)
    L = args.boxes ** 3
    order = low_discrepancy_ids(L, centre_leaf(args.boxes))
    steps = max(1, args.steps)
    pos = 0

    def take(k):
        nonlocal pos
        ids = [order[(pos + i) % L] for i in range(k)]
        pos += k
        return ids

    # warm-up steps: one leaf per worker each; the last one sizes the timed steps
    rate = None
    for _ in range(max(1, args.warmup)):
        ids = take(ref.workers)
        rate = len(ids) / ref.run(ids)
    per_step = max(ref.workers, int(round(rate * args.ref_seconds / steps / ref.workers)) * ref.workers)
    times, timed = [], 0
    for _ in range(steps):
        ids = take(per_step)
        times.append(ref.run(ids))
        timed += len(ids)
    total = float(sum(times))
    value = timed / total
    n, m = (args.p - 2) ** 3, 6 * (args.p - 2) ** 2
    from paper_2503_04033_b200.engine import dtn_flops
    config = config_of(args, world, L // world)
    config["sample_leaves"] = per_step
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / steps, "leaves_timed": timed,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config,
            "step": f"one step = DtN maps of {per_step} leaves drawn over the whole grid "
                    f"(bump-centre leaf first, golden-ratio sequence), the CPU analogue of the "
                    f"GPU step's {L // world} leaves",
            "fp64_tflops": value * dtn_flops(n, m) / 1e12,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": ref.workers, "kind": ref.kind,
                             "sample": f"{timed} leaves in {steps} steps, {ref.describe()}, {total:.1f} s"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# the GPU arm
# ---------------------------------------------------------------------------

def parity_check(out, pack, leaf_ids, tpl, fixture_name, k):
    """This run's maps vs the CPU oracle on ``k`` leaves spread over the share (the
    bump-centre and fixture leaves first) and vs the reference's own outputs where the
    share holds a fixture leaf (tests/golden/bench_cases.npz: T R for a probe R and
    sampled rows of T)."""
    from oracle import hps_oracle as O
    p = tpl.p
    boxes = int(round(1.0 / tpl.widths[0]))
    fx = {}
    if fixture_name and os.path.exists(FIXTURES):
        G = np.load(FIXTURES)
        for key in G.files:
            parts = key.split("/")
            if parts[0] == fixture_name and len(parts) == 3 and parts[2] == "dtn_R":
                idx = tuple(int(x) for x in parts[1].split("_"))
                fx[int(np.ravel_multi_index(idx, (boxes,) * 3))] = (
                    G[f"{parts[0]}/{parts[1]}/dtn_R"], G[f"{parts[0]}/R"],
                    G[f"{parts[0]}/{parts[1]}/dtn_rows_idx"], G[f"{parts[0]}/{parts[1]}/dtn_rows"])
    pos = {leaf: i for i, leaf in enumerate(leaf_ids)}
    chosen = spread_sample(leaf_ids, k, must=[centre_leaf(boxes)] + sorted(fx))
    otpl = O.OracleTemplate(tpl.widths, p)
    errs, ferrs, checked_fx = [], [], []
    for leaf in chosen:
        i = pos[leaf]
        got = out[i].cpu().numpy()
        ref, _, _ = O.leaf_dtn(otpl, pack[i, :3].T, None, pack[i, 3])
        errs.append(float(np.linalg.norm(got - ref) / np.linalg.norm(ref)))
        if leaf in fx:
            tR, R, rows, trow = fx[leaf]
            ferrs.append(max(float(np.linalg.norm(got @ R - tR) / np.linalg.norm(tR)),
                             float(np.linalg.norm(got[rows] - trow) / np.linalg.norm(trow))))
            checked_fx.append(leaf)
    res = {"checked_leaves": chosen, "max_rel_fro_err_vs_oracle": max(errs), "tolerance": TOL}
    if checked_fx:
        res["reference_fixture_leaves"] = checked_fx
        res["max_rel_err_vs_reference_fixture"] = max(ferrs)
    res["ok"] = max(errs + ferrs) <= TOL
    return res


def timed_dtn(eng, coeffs, out, stats, steps, warmup, local, barrier):
    """W untimed launches, then K launches bracketed by barrier + synchronize; CUDA
    events on the launching stream.  Returns (per-step ms list, wall s, clocks)."""
    import torch
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        eng.dtn(coeffs, out, stats, stream=stream)
    torch.cuda.synchronize()
    barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_wall = time.perf_counter()
        for k in range(steps):
            starts[k].record(stream)
            eng.dtn(coeffs, out, stats, stream=stream)
            ends[k].record(stream)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    barrier()
    return [s.elapsed_time(e) for s, e in zip(starts, ends)], t_wall, clk.summary()


def max_over_ranks(x, distributed, local):
    if not distributed:
        return x
    import torch
    t = torch.tensor([float(x)], device="cpu" if BACKEND == "gloo" else f"cuda:{local}",
                     dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def roofline(p, leaves, kernel_ms):
    from paper_2503_04033_b200.engine import dtn_flops_executed
    n, m = (p - 2) ** 3, 6 * (p - 2) ** 2
    achieved = leaves * dtn_flops_executed(n, m, p - 2) / (kernel_ms / 1e3) / 1e12
    per_leaf, src = traffic_per_leaf(p)
    return {"bound": "tensor", "achieved": achieved, "peak": PEAK_FP64_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / PEAK_FP64_TFLOPS,
            "traffic": per_leaf * leaves if per_leaf is not None else None,
            "kernel": "hps_leaf_kernel (assembly + LU + Schur, DMMA m8n8k4 f64)",
            "peak_source": "measured FP64 DMMA peak 37.1 TFLOP/s (cuBLAS DGEMM 35.5); "
                           "MEASURED_PEAKS.json has no FP64 entry",
            "traffic_source": (f"{src} (ncu --set full, DRAM bytes per leaf x leaves)" if src else
                               "no ncu capture at this order")}


def configs3_share(args, world, rank, local, distributed, barrier):
    """configs[3]: p = 20, 16^3 leaves, kappa = 80, 1/8 leaf-index share per GPU."""
    import torch
    from paper_2503_04033_b200.engine import LeafEngine
    c = CONFIGS3
    p, boxes, shards = c["p"], c["boxes"], c["shards"]
    share = rank % shards
    ids = shard_ids(boxes ** 3, shards, share)
    tpl, pack = make_shard(p, boxes, c["kappa"], leaf_ids=ids)
    L = len(ids)
    m = tpl.n_boundary
    eng = LeafEngine(tpl, False, True, device=local)
    coeffs = torch.from_numpy(pack).to(f"cuda:{local}")
    out = torch.empty((L, m, m), dtype=torch.float64, device=f"cuda:{local}")
    stats = torch.empty((L, 2), dtype=torch.float64, device=f"cuda:{local}")
    steps, warmup = args.configs3_steps, max(3, min(args.warmup, 3))
    step_ms, t_wall, clocks = timed_dtn(eng, coeffs, out, stats, steps, warmup, local, barrier)
    total_ms = max_over_ranks(float(sum(step_ms)), distributed, local)
    parity = parity_check(out, pack, ids, tpl, "c3_p20_bump_k80", 4) if rank == 0 else None
    del out, coeffs, stats, eng
    torch.cuda.empty_cache()
    value = world * L * steps / (total_ms / 1e3)
    return {"workload": f"3D variable-coefficient Helmholtz b(x), p={p}, {boxes}x{boxes}x{boxes} leaves, "
                        f"kappa={c['kappa']:g}, sharded across 8 GPUs by leaf index; rank r times "
                        f"share r ({L} leaves) — at N={world}, {world} of the 8 shares",
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": warmup, "ms_per_step": total_ms / steps, "leaves_per_gpu": L,
            "leaf_ids_rank0": [ids[0], ids[-1]],
            "l2": "outputs (%.1f GB) per GPU exceed the 126 MB L2" % (L * m * m * 8 / 1e9),
            "roofline": roofline(p, L, float(np.mean(step_ms))), "gpu_launches": steps,
            "parity": parity, "clocks": clocks, "wall_s_timed": t_wall}


def main(argv=None):
    args = parse(argv)
    if args.impl == "reference":
        reference_arm(args)
        return
    world, rank, local = dist_env()
    p, boxes = args.p, args.boxes
    n, m = (p - 2) ** 3, 6 * (p - 2) ** 2

    # CPU reference first, before pinned buffers and GPU work claim host resources
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(p, boxes, args.kappa, args.field, args.cpu_seconds)

    import torch
    torch.cuda.set_device(local)
    distributed = "RANK" in os.environ and "WORLD_SIZE" in os.environ  # launched by torchrun
    if distributed:
        import torch.distributed as dist
        # NCCL announces itself on stdout when the communicator is created; keep
        # stdout for the one JSON line (fd-level redirect: the print is native)
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            if BACKEND == "gloo":
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
            dist.barrier()
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)

    def barrier():
        if distributed:
            torch.distributed.barrier()

    from paper_2503_04033_b200.engine import LeafEngine, dtn_flops, dtn_flops_executed
    if args.leaves:
        leaf_ids = [k % boxes ** 3 for k in range(rank * args.leaves, (rank + 1) * args.leaves)]
    else:
        leaf_ids = shard_ids(boxes ** 3, world, rank)
    tpl, pack = make_shard(p, boxes, args.kappa, field=args.field, leaf_ids=leaf_ids)
    L = pack.shape[0]
    eng = LeafEngine(tpl, False, True, device=local)
    coeffs = torch.from_numpy(pack).to(f"cuda:{local}")
    out = torch.empty((L, m, m), dtype=torch.float64, device=f"cuda:{local}")
    stats = torch.empty((L, 2), dtype=torch.float64, device=f"cuda:{local}")
    step_ms, t_wall, clocks = timed_dtn(eng, coeffs, out, stats, args.steps, args.warmup, local, barrier)
    total_ms = max_over_ranks(float(sum(step_ms)), distributed, local)
    value = world * L * args.steps / (total_ms / 1e3)

    # parity of this run's output: 8 leaves per rank spread over the share (bump centre
    # first) vs the CPU oracle, and the reference's own outputs for fixture leaves
    fixture = {12: "c1_p12_const_k10", 16: "c2_p16_bump_k40"}.get(p) if boxes in (8, 16) else None
    if fixture == "c1_p12_const_k10" and (boxes != 8 or args.field != "const" or args.kappa != 10.0):
        fixture = None
    if fixture == "c2_p16_bump_k40" and (boxes != 16 or args.field != "bump" or args.kappa != 40.0):
        fixture = None
    parity = parity_check(out, pack, leaf_ids, tpl, fixture, 8 if world == 1 else 4)
    bad = max_over_ranks(0.0 if parity["ok"] else 1.0, distributed, local)
    parity["all_ranks_ok"] = bad == 0.0

    e2e = None
    if not args.no_e2e:
        # public API with HOST buffers: pinned coefficient input, pinned DtN output;
        # H2D of the coefficients and D2H of every DtN map inside the timed region.
        del out
        torch.cuda.empty_cache()
        chunk = eng.slots // 2   # D2H granularity of the single-launch streamed path
        # host memory: every rank of the node pins its coefficients and DtN maps
        # (p = 16: 45 GB per 16^3 leaves); cap the e2e batch to half of what the
        # node has available so a multi-GPU run cannot exhaust host RAM
        per_leaf = pack[0].nbytes + m * m * 8
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
        budget = 0.5 * host_mem_available() / max(local_world, 1)
        Le = L if L * per_leaf <= budget else max(chunk, int(budget // per_leaf) // chunk * chunk)
        Le = min(Le, L)
        h_coef = pinned_host((Le,) + pack.shape[1:])
        h_coef[:] = pack[:Le]
        h_out = pinned_host((Le, m, m))
        # untimed warm-up over the full batch: sizes the device streaming buffers
        eng.dtn_host(h_coef, out=h_out, chunk_leaves=chunk)
        barrier()
        ts = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            eng.dtn_host(h_coef, out=h_out, chunk_leaves=chunk)
            ts.append(time.perf_counter() - t0)
        e2e_t = max_over_ranks(float(np.mean(ts)), distributed, local)
        unpin_host(h_coef)
        unpin_host(h_out)
        del h_coef, h_out
        e2e = {"value": world * Le / e2e_t, "unit": UNIT, "leaves_per_gpu": Le,
               "h2d_bytes_per_step": int(Le * pack[0].nbytes), "d2h_bytes_per_step": int(Le * m * m * 8),
               "path": "LeafEngine.dtn_host -> hps_leaf_dtn_host (C ABI): H2D of all coefficients, "
                       "one persistent launch, D2H of each finished "
                       f"{chunk}-leaf chunk overlapped via device completion counters"}
    else:
        del out
    del coeffs, stats, eng
    torch.cuda.empty_cache()

    configs3 = None
    if args.configs3_steps > 0 and not args.leaves:
        configs3 = configs3_share(args, world, rank, local, distributed, barrier)

    if rank == 0:
        flops_ref = dtn_flops(n, m)
        flops_leaf = dtn_flops_executed(n, m, p - 2)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_of(args, world, L),
            "fp64_tflops": value * flops_leaf / 1e12,
            "fp64_tflops_reference_equivalent": value * flops_ref / 1e12,
            "flops_per_leaf": flops_leaf,
            "flops_per_leaf_reference_algorithm": flops_ref,
            "roofline": roofline(p, L, float(np.mean(step_ms))),
            "gpu_launches": args.steps,
            "e2e": e2e, "cpu_baseline": cpu, "parity": parity,
            "clocks": clocks, "wall_s_timed": t_wall,
            "configs3": configs3,
        }
        print(json.dumps(line), flush=True)
    if distributed:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
