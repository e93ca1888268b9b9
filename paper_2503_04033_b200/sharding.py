"""Leaf sharding across GPUs (one process per GPU, torch.distributed).

Leaf boxes are independent, so the build stage splits them by leaf index
into contiguous shards, one per rank; every rank reduces its shard on its own
GPU with no collective on the data path.  The only exchange is the return of
the finished DtN blocks to the rank that owns the host-side sparse assembly
and factorization (paper §3.2: DtNs are "transferred collectively to the
CPU"), done once per flush with a gather — or, with the interface assembly
on the device (``sharded_interface``), one sum-reduce of each rank's partial
CSR values of T and C, which carries nnz(T) + nnz(C) doubles instead of every
m x m map and leaves root nothing to scatter.
"""

from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np


def shard_range(n_leaves: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced [start, stop) of leaf ids owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(n_leaves, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def max_over_ranks(value: float) -> float:
    """Slowest rank's time: the multi-GPU timing rule (max over ranks)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_to_root(ids: Sequence[int], blocks: np.ndarray, root: int = 0
                   ) -> Optional[List[Tuple[np.ndarray, np.ndarray]]]:
    """Gather (leaf ids, DtN blocks) of every rank on ``root``; None elsewhere."""
    import torch.distributed as dist
    payload = (np.asarray(ids, dtype=np.int64), np.ascontiguousarray(blocks))
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [payload]
    out = [None] * dist.get_world_size() if dist.get_rank() == root else None
    dist.gather_object(payload, out, dst=root)
    return out


def sharded_dtn(disc, coeffs, world: int, rank: int,
                compute: Optional[Callable[[np.ndarray], np.ndarray]] = None,
                template=None, root: int = 0):
    """DtN maps of this rank's leaf shard, gathered on ``root`` in leaf order.

    ``compute`` maps a coefficient pack (L, ncoef, n) to DtN blocks (L, m, m);
    by default the rank's GPU engine.  Returns the (n_leaves, m, m) array on
    ``root`` and None on the other ranks.
    """
    from .local_ops import LeafTemplate, check_pivots, pack_coefficients
    start, stop = shard_range(len(disc.leaves), world, rank)
    ids = list(range(start, stop))
    template = template or LeafTemplate(disc.leaf_widths, disc.p, disc.corner_mode,
                                        coeffs.has_cross_terms)
    if compute is None:
        from .engine import LeafEngine
        import torch
        eng = LeafEngine.for_template(template, coeffs, device=torch.cuda.current_device())

        def compute(pack):
            dtn, stats = eng.dtn_host(pack)
            check_pivots(stats, [disc.leaves[i].index for i in ids])
            return dtn
    m = template.n_boundary
    if ids:
        from .condensation import interior_points
        blocks = compute(pack_coefficients(coeffs, interior_points(disc, ids), len(ids)))
    else:
        blocks = np.empty((0, m, m))
    parts = gather_to_root(ids, blocks, root)
    if parts is None:
        return None
    out = np.empty((len(disc.leaves), m, m))
    for part_ids, part_blocks in parts:
        out[part_ids] = part_blocks
    return out


def sharded_interface(disc, coeffs, world: int, rank: int, root: int = 0, pattern=None,
                      compute: Optional[Callable[[np.ndarray], np.ndarray]] = None,
                      scatter: Optional[Callable] = None, template=None):
    """T and the Dirichlet coupling C, assembled from every rank's leaf shard.

    Each rank reduces its shard and adds the DtN maps into its own partial CSR
    values of T and C (``hps_interface_scatter`` on its GPU); one sum-reduce
    of the value arrays onto ``root`` is the only exchange.  An entry of T has
    at most two nonzero partials and x + 0 = x, so the result is bit-identical
    to a single-process assembly.  ``compute`` / ``scatter`` replace the
    rank's GPU (pack -> DtN maps; (pattern, maps, ids) -> (t_vals, c_vals))
    for CPU tests.  Returns (T, C) on root, None elsewhere.
    """
    import torch
    import torch.distributed as dist
    from .assembly import DeviceAssembler, pattern_for
    from .condensation import interior_points
    from .local_ops import LeafTemplate, check_pivots, pack_coefficients
    pattern = pattern or pattern_for(disc)
    start, stop = shard_range(len(disc.leaves), world, rank)
    ids = list(range(start, stop))
    pack = pack_coefficients(coeffs, interior_points(disc, ids), len(ids)) if ids else None
    if compute is None:
        from .engine import LeafEngine
        template = template or LeafTemplate(disc.leaf_widths, disc.p, disc.corner_mode,
                                            coeffs.has_cross_terms)
        device = torch.cuda.current_device()
        asm = DeviceAssembler(pattern, device)
        if ids:
            eng = LeafEngine.for_template(template, coeffs, device=device)
            dtn, stats = eng.dtn(pack)
            check_pivots(stats.cpu().numpy(), [disc.leaves[i].index for i in ids])
            asm.add(dtn, ids)
        vals = [asm.t_vals[:pattern.nnz[0]], asm.c_vals[:pattern.nnz[1]]]
    else:
        if ids:
            t_vals, c_vals = scatter(pattern, compute(pack), ids)
        else:
            t_vals, c_vals = np.zeros(pattern.nnz[0]), np.zeros(pattern.nnz[1])
        vals = [torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)) for v in (t_vals, c_vals)]
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        for v in vals:
            dist.reduce(v, dst=root, op=dist.ReduceOp.SUM)
        if dist.get_rank() != root:
            return None
    return pattern.matrices(vals[0].cpu().numpy(), vals[1].cpu().numpy())
