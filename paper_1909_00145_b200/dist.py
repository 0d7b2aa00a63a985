"""Multi-GPU plumbing for the CSC hot path: one process per GPU, images sharded.

Codes are independent per image ("computing sparse codes is a
data-independent process"); the mask is a counter-based function of (seed, t,
k, u, v), identical on every rank without communication (reading R5).  The
images of a batch are split in contiguous blocks; the filters are replicated.
The library (csc_filter_step / csc_objective) all-reduces the filter gradient,
||Zg||^2 and the objective parts with NCCL on its own stream; this module only
does the bootstrap: rank partition and the ncclUniqueId broadcast over
torch.distributed (PyTorch is plumbing here).
"""
from __future__ import annotations

import os
from typing import Optional, Tuple


def env_rank() -> Tuple[int, int, int]:
    """(world, rank, local_rank) from the torchrun environment (1, 0, 0 when absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block [n0, n1) of n images owned by `rank` (sizes differ by at most one)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("need world >= 1 and 0 <= rank < world")
    return (rank * n) // world, ((rank + 1) * n) // world


def broadcast_nccl_id(group=None, device=None) -> bytes:
    """Rank 0 creates an ncclUniqueId through the C ABI (csc_nccl_unique_id); every rank
    returns the same 128 bytes.  Works with an NCCL (CUDA tensor) or gloo (CPU tensor) group."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                             if backend == "nccl" else torch.device("cpu"))
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        from . import nccl_unique_id
        buf.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast(buf, src, group=group)
    return bytes(buf.cpu().numpy().tobytes())


def sharded_context(n_images: int, K: int, s: int, H: int, W: int, *, device: Optional[int] = None,
                    stream=None, group=None):
    """Create this rank's Context for a batch of n_images sharded over the default group.
    Returns (ctx, (n0, n1)).  Collective: every rank must call it."""
    import torch.distributed as dist

    from . import Context
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n0, n1 = shard(n_images, world, rank)
    nid = broadcast_nccl_id(group) if world > 1 else None
    ctx = Context(n1 - n0, K, s, H, W, world=world, rank=rank, device=device, stream=stream, nccl_id=nid)
    return ctx, (n0, n1)
