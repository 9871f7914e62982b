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


def gather_rows(rows, device="cpu"):
    """All-gather a rank's 2-D int32 array (variable row count) -> every rank's
    rows concatenated in rank order (numpy).  One size exchange, then one
    all_gather of row blocks padded to the longest (NCCL: pass device="cuda").
    Returns the input when not distributed."""
    import numpy as np
    import torch
    import torch.distributed as dist

    rows = np.ascontiguousarray(rows, dtype=np.int32)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return rows
    world = dist.get_world_size()
    width = rows.shape[1]
    n = torch.tensor([rows.shape[0]], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(s.item()) for s in sizes]
    cap = max(max(sizes), 1)
    mine = torch.zeros((cap, width), dtype=torch.int32, device=device)
    if rows.shape[0]:
        mine[:rows.shape[0]] = torch.from_numpy(rows).to(device)
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    return np.concatenate([p[:s].cpu().numpy() for p, s in zip(parts, sizes)], axis=0)


def allgather_concat(local, device="cpu"):
    """All-gather a rank's 1-D tensor of any length -> every rank's pieces
    concatenated in rank order, as a tensor on ``local``'s device.  One size
    exchange, then one all_gather of pieces padded to the longest (the
    collective runs on ``device``: "cpu" for gloo, the rank's GPU for NCCL).
    Returns ``local`` when not distributed."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    world = dist.get_world_size()
    n = torch.tensor([local.numel()], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(v.item()) for v in sizes]
    cap = max(max(sizes), 1)
    mine = torch.zeros(cap, dtype=local.dtype, device=device)
    if local.numel():
        mine[:local.numel()] = local.to(device)
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    return torch.cat([q[:k] for q, k in zip(parts, sizes)]).to(local.device)


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


def balanced_match(match_local, origins, device="cpu"):
    """One level of the re-balanced range sharding: every rank holds the same
    global range list ``origins`` (int32 [M, 2]); rank r matches the
    contiguous share slab_for_rank(M, r, world) with ``match_local(share) ->
    (err int64, idx int64, rmean float64)`` and the shares are all-gathered
    in rank order, so every rank continues with the whole level's result
    (and so the same next-level list).  Re-slicing per level keeps the ranks
    balanced whatever the data-dependent splits were."""
    import numpy as np
    import torch.distributed as dist

    o = np.asarray(origins, dtype=np.int32).reshape(-1, 2)
    dist_on = dist.is_available() and dist.is_initialized()
    world = dist.get_world_size() if dist_on else 1
    rank = dist.get_rank() if dist_on else 0
    lo, hi = slab_for_rank(o.shape[0], rank, world)
    rows = np.zeros((hi - lo, 6), dtype=np.int32)
    if hi > lo:
        err, idx, rmean = match_local(o[lo:hi])
        rows[:, 0:2] = np.ascontiguousarray(err, dtype=np.int64).view(np.int32).reshape(-1, 2)
        rows[:, 2:4] = np.ascontiguousarray(idx, dtype=np.int64).view(np.int32).reshape(-1, 2)
        rows[:, 4:6] = np.ascontiguousarray(rmean, dtype=np.float64).view(np.int32).reshape(-1, 2)
    full = gather_rows(rows, device=device)
    return (np.ascontiguousarray(full[:, 0:2]).view(np.int64).reshape(-1),
            np.ascontiguousarray(full[:, 2:4]).view(np.int64).reshape(-1),
            np.ascontiguousarray(full[:, 4:6]).view(np.float64).reshape(-1))
