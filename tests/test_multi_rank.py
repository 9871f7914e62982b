"""Multi-rank (world size 2, gloo on CPU) coverage of the sharding and the
timing reduction bench.py uses under torchrun."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1502_00324_b200 import sharding


def test_images_and_slabs_partition_the_work():
    for world in (1, 2, 3, 4, 8):
        imgs = sorted(i for r in range(world) for i in sharding.images_for_rank(64, r, world))
        assert imgs == list(range(64))
        slabs = [sharding.slab_for_rank(1024, r, world) for r in range(world)]
        assert slabs[0][0] == 0 and slabs[-1][1] == 1024
        assert all(a[1] == b[0] for a, b in zip(slabs, slabs[1:]))
        assert max(b - a for a, b in slabs) - min(b - a for a, b in slabs) <= 1
    with pytest.raises(ValueError):
        sharding.images_for_rank(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = sharding.images_for_rank(64, rank, world)
    metrics = dict(step_ms_total=10.0 * (rank + 1), e2e_s_total=1.0 + rank, kernel_ms_total=3.0 - rank,
                   comparisons=1000 * len(mine), pixels=512 * 512 * len(mine), alg_ops=7 * (rank + 1))
    out = sharding.reduce_metrics(metrics)
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_reduce_metrics_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in (0, 1):
        out = results[rank]
        assert out["step_ms_total"] == 20.0          # max over ranks
        assert out["e2e_s_total"] == 2.0
        assert out["kernel_ms_total"] == 3.0
        assert out["comparisons"] == 64 * 1000       # sum over ranks = whole job
        assert out["pixels"] == 64 * 512 * 512
        assert out["alg_ops"] == 21


def _gather_worker(rank, world, port, q):
    import numpy as np
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank r contributes r + 2 records (one rank may be empty in general)
    rows = np.arange((rank + 2) * 6, dtype=np.int32).reshape(-1, 6) + 1000 * rank
    out = sharding.gather_rows(rows)
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_rows_gloo_world2_rank_order():
    """The record all-gather of encode_distributed: variable row counts,
    concatenated in rank order on every rank (gloo, world size 2)."""
    import numpy as np

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.concatenate([np.arange((r + 2) * 6, dtype=np.int32).reshape(-1, 6) + 1000 * r
                           for r in range(2)])
    for rank in (0, 1):
        assert np.array_equal(results[rank], want)


def test_bench_gpus2_spawns_two_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself as two ranks
    (torch.distributed.run on 127.0.0.1); with the CPU arm, rank 0 prints the
    one JSON line and rank 1 exits 0 without work."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--workload", "c1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0


def _fake_match(share):
    """Deterministic stand-in for ctx.match_level: (err, idx, rmean) per origin."""
    import numpy as np

    s = np.asarray(share, dtype=np.int64).reshape(-1, 2)
    return s[:, 0] * 7 + s[:, 1], s[:, 0] + 3 * s[:, 1] + (1 << 40), s[:, 0] / 2.0 + s[:, 1] / 3.0


def _balanced_worker(rank, world, port, q):
    import numpy as np
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = []

    def local(share):
        calls.append(len(share))
        return _fake_match(share)

    results = []
    for m in (0, 1, 5, 1024, 1027):  # a level's range count, split unevenly by the quadtree
        o = np.stack([np.arange(m) % 97, np.arange(m) // 97], axis=1).astype(np.int32)
        results.append(sharding.balanced_match(local, o))
    q.put((rank, results, calls))
    dist.barrier()
    dist.destroy_process_group()


def test_balanced_match_gloo_world2():
    """Per-level re-balancing: each rank matches an even share of the level's
    ranges and every rank gets the whole level's (err, idx, mean), in order."""
    import numpy as np

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_balanced_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {r: (res, calls) for r, res, calls in (q.get(timeout=120) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k, m in enumerate((0, 1, 5, 1024, 1027)):
        o = np.stack([np.arange(m) % 97, np.arange(m) // 97], axis=1).astype(np.int32)
        want = _fake_match(o)
        for rank in (0, 1):
            res = got[rank][0][k]
            for a, b in zip(res, want):
                assert np.array_equal(a, b)
    # each rank matched exactly its even share of every level (empty shares skip the call)
    for rank in (0, 1):
        want = [hi - lo for lo, hi in (sharding.slab_for_rank(m, rank, 2)
                                       for m in (0, 1, 5, 1024, 1027)) if hi > lo]
        assert got[rank][1] == want


def _concat_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # the sharded pool build's exchanges: a row slice of every window's
    # entropy (contiguous, concatenates in rank order) and a variable-length
    # survivor list (rank 1 may hold none)
    ny, nx = 7, 5
    lo, hi = sharding.slab_for_rank(ny, rank, world)
    full = torch.arange(ny * nx, dtype=torch.float64) * 0.5
    ent = sharding.allgather_concat(full[lo * nx:hi * nx].clone())
    keys = torch.arange(3 * (1 - rank), dtype=torch.int64) + 100 * rank
    got = sharding.allgather_concat(keys)
    q.put((rank, bool(torch.equal(ent, full)), got.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_allgather_concat_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_concat_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {r[0]: r[1:] for r in (q.get(timeout=120) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in (0, 1):
        same, got = res[rank]
        assert same and got == [0, 1, 2]
