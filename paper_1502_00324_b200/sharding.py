"""Work sharding across ranks (one process per GPU) and the timing reduction.

The encoder search shards without any data-path exchange:
images of a batch are independent, and so are the top-level 16x16 range
slots of one image given the replicated pool (codec.py:134-142).  The only
collective is the final reduction of per-rank timings and counters: times
take the MAX over ranks (the job finishes with the slowest rank), counters
the SUM.
"""

from __future__ import annotations


def images_for_rank(n_images: int, rank: int, world: int) -> list:
    """Round-robin image indices of a batch for one rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    return list(range(rank, n_images, world))


def slab_for_rank(n_items: int, rank: int, world: int) -> tuple:
    """Contiguous [start, stop) slab of n_items for one rank (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


MAX_KEYS = ("step_ms_total", "e2e_s_total", "kernel_ms_total")
SUM_KEYS = ("comparisons", "pixels", "alg_ops")


def reduce_metrics(metrics: dict, device="cpu") -> dict:
    """All-reduce a rank's metrics: MAX for times, SUM for counters.

    Works with any initialised torch.distributed backend (nccl on the GPU
    box, gloo in the CPU tests); returns the input unchanged when not
    distributed.
    """
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return dict(metrics)
    mx = torch.tensor([float(metrics[k]) for k in MAX_KEYS], dtype=torch.float64, device=device)
    sm = torch.tensor([float(metrics[k]) for k in SUM_KEYS], dtype=torch.float64, device=device)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    out = dict(metrics)
    out.update({k: float(v) for k, v in zip(MAX_KEYS, mx.tolist())})
    out.update({k: float(v) for k, v in zip(SUM_KEYS, sm.tolist())})
    return out
