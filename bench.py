"""Leaf DtN throughput on B200: the two-level HPS solver's batched leaf-box reduction.

Workload (BASELINE.json configs[2]): 3D variable-coefficient Helmholtz
    -Lap u - kappa^2 b(x) u,  b(x) = 1 - 0.5 exp(-|x - c|^2 / (2 * 0.15^2)),
p = 16 Chebyshev nodes per axis, 16 x 16 x 16 leaf boxes per GPU, kappa = 40.
One step = the DtN maps of every leaf of the rank's shard (operator assembly,
pivoted LU of A_ii, Schur complement), inputs resident in HBM.  Under torchrun
each rank owns its own 16^3-leaf slab of a 16 x 16 x 16N leaf grid (weak
scaling, no collective on the data path).

Prints ONE JSON line (rank 0).  ``--impl reference`` times the reference's CPU
algorithm (the numpy/LAPACK oracle port in oracle/) on the host cores instead.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAK_FP64_TFLOPS = 37.1   # measured DMMA issue peak, profiles/r01_fp64_probe_dmma_dfma.log
PEAK_FP64_CUBLAS = 35.5   # measured cuBLAS DGEMM, profiles/r01_fp64_probe_cublas_cusolver.log


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--p", type=int, default=16)
    ap.add_argument("--boxes", type=int, default=16, help="leaf boxes per axis per GPU")
    ap.add_argument("--kappa", type=float, default=40.0)
    ap.add_argument("--field", default="bump", choices=["bump", "const"],
                    help="bump: variable-coefficient b(x) (configs 2-3); const: b = 1 (configs[1])")
    ap.add_argument("--leaves", type=int, default=0, help="override leaves per rank (profiling)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=60.0,
                    help="reference arm: total CPU seconds over warmup + timed steps")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
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


def make_shard(p, boxes, kappa, rank, world, leaves_override=0, field="bump"):
    """Coefficient packs (L, 4, n) for this rank's slab of the unit-cube-stacked leaf grid.
    field "bump": -Lap u - kappa^2 b(x) u (configs 2-3); "const": b = 1 (configs[1])."""
    from paper_2503_04033_b200.local_ops import LeafTemplate
    h = 1.0 / boxes
    tpl = LeafTemplate((h, h, h), p, "drop", False)
    L = leaves_override or boxes ** 3
    n = tpl.n_interior
    inner = tpl.ref_offsets[1:-1]
    pack = np.empty((L, 4, n))
    pack[:, :3, :] = 1.0
    idx = np.array(list(np.ndindex(boxes, boxes, boxes)))[:L] if L <= boxes ** 3 else \
        np.array([np.unravel_index(k % boxes ** 3, (boxes,) * 3) for k in range(L)])
    idx = idx.astype(float)
    idx[:, 2] += rank * boxes
    for k0 in range(0, L, 256):
        lo = idx[k0:k0 + 256] * h
        B = len(lo)
        g = [lo[:, a, None] + h * inner[None, :] for a in range(3)]
        q = len(inner)
        X = np.broadcast_to(g[0][:, :, None, None], (B, q, q, q))
        Y = np.broadcast_to(g[1][:, None, :, None], (B, q, q, q))
        Z = np.broadcast_to(g[2][:, None, None, :], (B, q, q, q))
        pts = np.stack([X, Y, Z], axis=-1).reshape(-1, 3)
        b = bump_b(pts) if field == "bump" else np.ones(len(pts))
        pack[k0:k0 + B, 3, :] = (-kappa * kappa * b).reshape(B, n)
    return tpl, pack


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
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = [nm for i, nm in enumerate(names) if any(r[3 + i] == "Active" for r in rows)]
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())}


def traffic_per_launch(leaves):
    """DRAM bytes per launch from the committed ncu --set full capture (per-leaf, scaled)."""
    path = os.path.join(ROOT, "profiles", "r01_ncu_summary.json")
    try:
        per_leaf = json.load(open(path))["traffic_bytes_per_leaf"]
    except (OSError, KeyError, ValueError):
        return None
    return per_leaf * leaves


def blas_threads():
    """Threads the host BLAS (OpenBLAS under numpy/scipy) actually uses."""
    try:
        from threadpoolctl import threadpool_info
        n = [i["num_threads"] for i in threadpool_info() if i.get("user_api") == "blas"]
        if n:
            return int(max(n))
    except Exception:
        pass
    return os.cpu_count() or 1


def cpu_reference(tpl, pack, seconds, steps=1):
    """The reference's CPU algorithm (oracle port of local_ops.build_leaf_factors) on host cores."""
    from oracle import hps_oracle as O
    otpl = O.OracleTemplate(tpl.widths, tpl.p)
    cores = blas_threads()
    times, done = [], 0
    t_start = time.perf_counter()
    for _ in range(steps):
        t0 = time.perf_counter()
        k = 0
        while True:
            c = pack[(done + k) % pack.shape[0]]
            O.leaf_dtn(otpl, c[:3].T, None, c[3])
            k += 1
            if time.perf_counter() - t0 >= seconds and k >= 2:
                break
        done += k
        times.append((time.perf_counter() - t0) / k)
    per_leaf = float(np.median(times))
    return {"value": 1.0 / per_leaf, "unit": "leaf DtN maps/s", "cores": cores, "kind": "port",
            "sample": f"{done} leaves of the workload (p={tpl.p}), numpy/scipy LAPACK getrf+getrs+gemm "
                      f"with OpenBLAS on {cores} host threads, {time.perf_counter() - t_start:.1f} s"}


def main():
    args = parse()
    world, rank, local = dist_env()
    p, boxes = args.p, args.boxes
    leaves_per_gpu = args.leaves or boxes ** 3
    grid = (f"{boxes}x{boxes}x{boxes} leaves per GPU" if leaves_per_gpu == boxes ** 3 else
            f"{leaves_per_gpu} leaves per GPU (a 1/{boxes ** 3 // max(leaves_per_gpu, 1)} shard of a "
            f"{boxes}x{boxes}x{boxes} leaf grid)")
    kind = ("3D variable-coefficient Helmholtz b(x) (Gaussian bump)" if args.field == "bump"
            else "3D constant-coefficient Helmholtz")
    workload = (f"{kind}, p={p}, {grid}, "
                f"kappa={args.kappa:g}")
    n = (p - 2) ** 3
    m = 6 * (p - 2) ** 2
    from paper_2503_04033_b200.engine import dtn_flops, dtn_flops_executed
    flops_ref = dtn_flops(n, m)                     # the reference's dense algorithm
    flops_leaf = dtn_flops_executed(n, m, p - 2)    # what the kernel executes
    metric = "leaf DtN maps/sec"

    if args.impl == "reference":
        if rank != 0:
            return
        tpl, pack = make_shard(p, boxes, args.kappa, 0, 1, leaves_override=min(64, boxes ** 3),
                               field=args.field)
        steps = max(1, args.steps)
        per_step = max(min(2.0, args.ref_seconds), args.ref_seconds / (steps + args.warmup))
        for _ in range(args.warmup):
            cpu_reference(tpl, pack, seconds=min(per_step, 2.0))
        base = cpu_reference(tpl, pack, seconds=per_step, steps=steps)
        line = {"metric": metric, "value": base["value"], "unit": "leaf DtN maps/s", "impl": "reference",
                "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * leaves_per_gpu / base["value"], "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload, "p": p, "leaves_per_gpu": leaves_per_gpu,
                           "kappa": args.kappa, "step": "bounded CPU sample of the workload"},
                "fp64_tflops": base["value"] * flops_ref / 1e12,
                "cpu_baseline": base,
                "e2e": {"value": base["value"], "unit": "leaf DtN maps/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    # CPU reference first, before pinned buffers and GPU work claim host resources
    cpu = None
    if rank == 0 and not args.no_cpu:
        tpl0, pack0 = make_shard(p, boxes, args.kappa, 0, 1, min(64, boxes ** 3), field=args.field)
        cpu = cpu_reference(tpl0, pack0, seconds=args.cpu_seconds)

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
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
            dist.barrier()
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)
    from paper_2503_04033_b200.engine import LeafEngine

    tpl, pack = make_shard(p, boxes, args.kappa, rank, world, args.leaves, field=args.field)
    L = pack.shape[0]
    eng = LeafEngine(tpl, False, True, device=local)
    coeffs = torch.from_numpy(pack).to(f"cuda:{local}")
    out = torch.empty((L, m, m), dtype=torch.float64, device=f"cuda:{local}")
    stats = torch.empty((L, 2), dtype=torch.float64, device=f"cuda:{local}")
    stream = torch.cuda.current_stream()

    def barrier():
        if distributed:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        eng.dtn(coeffs, out, stats)
    torch.cuda.synchronize()
    barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_wall = time.perf_counter()
        for k in range(args.steps):
            starts[k].record(stream)
            eng.dtn(coeffs, out, stats)
            ends[k].record(stream)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = float(sum(step_ms))
    if distributed:
        t = torch.tensor([total_ms], device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    value = world * L * args.steps / (total_ms / 1e3)
    kernel_ms = float(np.mean(step_ms))
    achieved = L * flops_leaf / (kernel_ms / 1e3) / 1e12

    # parity spot check of this run's output against the CPU oracle (2 leaves)
    parity = None
    if rank == 0:
        from oracle import hps_oracle as O
        otpl = O.OracleTemplate(tpl.widths, p)
        errs = []
        for k in (0, L - 1):
            ref, _, _ = O.leaf_dtn(otpl, pack[k, :3].T, None, pack[k, 3])
            got = out[k].cpu().numpy()
            errs.append(float(np.linalg.norm(got - ref) / np.linalg.norm(ref)))
        parity = {"checked_leaves": 2, "max_rel_fro_err_vs_oracle": max(errs), "tolerance": 1e-10}

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
        e2e_t = float(np.mean(ts))
        if distributed:
            t = torch.tensor([e2e_t], device=f"cuda:{local}", dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e2e_t = float(t.item())
        unpin_host(h_coef)
        unpin_host(h_out)
        del h_coef, h_out
        e2e = {"value": world * Le / e2e_t, "unit": "leaf DtN maps/s", "leaves_per_gpu": Le,
               "h2d_bytes_per_step": int(Le * pack[0].nbytes), "d2h_bytes_per_step": int(Le * m * m * 8),
               "path": "LeafEngine.dtn_host -> hps_leaf_dtn_host (C ABI): H2D of all coefficients, "
                       "one persistent launch, D2H of each finished "
                       f"{chunk}-leaf chunk overlapped via device completion counters"}


    if rank == 0:
        line = {
            "metric": metric, "value": value, "unit": "leaf DtN maps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": workload, "p": p, "leaves_per_gpu": L, "n_interior": n,
                       "n_boundary": m, "kappa": args.kappa,
                       "l2": "inputs (coefficients %.0f MB) and outputs (%.1f GB) exceed the 126 MB L2"
                             % (pack.nbytes / 1e6, L * m * m * 8 / 1e9),
                       "parallelism": f"leaf-sharded x{world}, no data-path collective"},
            "fp64_tflops": value * flops_leaf / 1e12,
            "fp64_tflops_reference_equivalent": value * flops_ref / 1e12,
            "flops_per_leaf": flops_leaf,
            "flops_per_leaf_reference_algorithm": flops_ref,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": PEAK_FP64_TFLOPS,
                         "unit": "TFLOP/s", "frac": achieved / PEAK_FP64_TFLOPS,
                         "traffic": traffic_per_launch(L),
                         "kernel": "hps_leaf_kernel (assembly + LU + Schur, DMMA m8n8k4 f64)",
                         "peak_source": "measured FP64 DMMA peak 37.1 TFLOP/s (cuBLAS DGEMM 35.5); "
                                        "MEASURED_PEAKS.json has no FP64 entry",
                         "traffic_source": "profiles/r01_ncu_summary.json (ncu --set full, per leaf x leaves)"},
            "gpu_launches": args.steps,
            "e2e": e2e, "cpu_baseline": cpu, "parity": parity,
            "clocks": clk.summary(), "wall_s_timed": t_wall,
        }
        print(json.dumps(line), flush=True)
    if distributed:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
