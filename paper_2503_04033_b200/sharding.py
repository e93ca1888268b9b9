"""Leaf sharding across GPUs (one process per GPU, torch.distributed).

Leaf boxes are independent, so every stage of the solver splits them by leaf
index into contiguous shards, one per rank, and every rank reduces its shard
on its own GPU with no collective on the data path (the reference's worker
pool over leaves, condensation.py:248-264, 325-333, 385-391, becomes one
process per GPU).  The exchanges are off the leaf path and happen once per
stage:

* ``build``        — each rank scatters its maps into its own partial CSR values
                     of T and C on its GPU; one sum-reduce of those arrays onto
                     the root, which factorizes (``reduce_sum_to_root``);
* ``reduce_load``  — the same for the interface right-hand side g_b;
* ``solve``        — the root's boundary solution goes to every rank
                     (``broadcast_from_root``), each rank solves its leaves'
                     interiors, the interior values come back to the root
                     (``gather_rows_to_root``), and the assembled solution is
                     broadcast so every rank returns the same report.

Sums are bit-identical to one process: an entry of T or g_b has at most two
nonzero contributions and x + 0 = x, x + y = y + x in IEEE arithmetic.
Collectives run on the GPU tensors under NCCL and on CPU copies under gloo
(gloo has no CUDA reduce).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np


def shard_range(n_leaves: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced [start, stop) of leaf ids owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(n_leaves, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


@dataclass(frozen=True)
class Shard:
    """This process's place in a multi-rank solve."""
    world: int
    rank: int
    root: int
    start: int
    stop: int

    @property
    def is_root(self) -> bool:
        return self.rank == self.root

    @property
    def ids(self):
        return range(self.start, self.stop)


def current_shard(n_leaves: int, enabled: Optional[bool] = None, root: int = 0) -> Optional[Shard]:
    """The rank's leaf shard when torch.distributed is initialized with more than
    one rank (and ``enabled`` is not False); None for a single-process solve."""
    if enabled is False:
        return None
    try:
        import torch.distributed as dist
    except ImportError:
        return None
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return None
    world, rank = dist.get_world_size(), dist.get_rank()
    start, stop = shard_range(n_leaves, world, rank)
    return Shard(world, rank, root, start, stop)


def _backend_device(tensor):
    """Where a collective on ``tensor`` runs: its GPU under NCCL, the CPU otherwise."""
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        if tensor.device.type != "cuda":
            return tensor.to(f"cuda:{torch.cuda.current_device()}")
        return tensor
    return tensor.cpu() if tensor.device.type != "cpu" else tensor


def reduce_sum_to_root(tensor, root: int = 0) -> Optional[np.ndarray]:
    """Element-wise sum over ranks of a float64 tensor (device or host), as numpy on
    ``root``; None elsewhere.  The tensor may be reduced in place."""
    import torch.distributed as dist
    t = _backend_device(tensor.contiguous())
    dist.reduce(t, dst=root, op=dist.ReduceOp.SUM)
    return t.cpu().numpy() if dist.get_rank() == root else None


def broadcast_from_root(array: Optional[np.ndarray], n: int, root: int = 0) -> np.ndarray:
    """The root's float64 vector of length ``n`` on every rank."""
    import torch
    import torch.distributed as dist
    if dist.get_rank() == root:
        t = torch.from_numpy(np.ascontiguousarray(array, dtype=np.float64))
    else:
        t = torch.empty(n, dtype=torch.float64)
    t = _backend_device(t)
    dist.broadcast(t, src=root)
    return t.cpu().numpy()


def gather_rows_to_root(rows: np.ndarray, counts, root: int = 0) -> Optional[np.ndarray]:
    """Concatenate every rank's (count_r, w) float64 rows in rank order on ``root``
    (counts = rows per rank, known everywhere); None elsewhere."""
    import torch
    import torch.distributed as dist
    width = rows.shape[1] if rows.ndim == 2 else 0
    cap = max(counts) if counts else 0
    buf = torch.zeros((cap, width), dtype=torch.float64)
    if len(rows):
        buf[:len(rows)] = torch.from_numpy(np.ascontiguousarray(rows, dtype=np.float64))
    buf = _backend_device(buf)
    world = dist.get_world_size()
    if dist.get_rank() == root:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.gather(buf, parts, dst=root)
        return np.concatenate([p[:c].cpu().numpy() for p, c in zip(parts, counts)])
    dist.gather(buf, None, dst=root)
    return None


def max_over_ranks(value: float) -> float:
    """Slowest rank's time: the multi-GPU timing rule (max over ranks)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = _backend_device(torch.tensor([float(value)], dtype=torch.float64))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
