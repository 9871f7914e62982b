"""Range-sharded encode across two processes on the one GPU of
the test box: two ranks with their own contexts on cuda:0, a gloo process
group (the code path is the one torchrun + NCCL runs on an 8-GPU node: the
pool's entropy pass sharded by window rows and all-gathered, the replicated
ranking, a slab of ranges per rank, one record all-gather).  The ranks' kernels never
wait on each other, so sharing a GPU is safe."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_1502_00324_b200 as fc
    from paper_1502_00324_b200 import _native

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = np.load(os.path.join(GOLDEN, "encode_c2.npz"))
    caps = tuple(int(v) for v in g["caps_c2"])
    params = fc.PoolParams(pool_cap=max(caps), strides=tuple(int(v) for v in g["strides_c2"]),
                           level_caps=caps)
    cfg = fc.EncoderConfig(pool=params, thresholds=tuple(float(v) for v in g["thresholds_c2"]))
    ctx = _native.Context(0)
    stream, report = fc.encode_distributed(fc.GrayImage(g["image_c2"]), cfg, context=ctx)
    rec, _, stats = fc.encode_shard(fc.GrayImage(g["image_c2"]), cfg, rank, world, context=ctx)
    q.put((rank, fc.serialize(stream) == g["bytes_c2"].tobytes(), int(report.collage_ssd),
           int(report.comparisons), sum(s["comparisons"] for s in stats), rec.shape[0]))
    dist.barrier()
    dist.destroy_process_group()


def test_encode_distributed_two_processes_c2_bytes():
    g = np.load(os.path.join(GOLDEN, "encode_c2.npz"))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {r[0]: r[1:] for r in (q.get(timeout=600) for _ in procs)}
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank in (0, 1):
        same, collage, comps, _, _ = res[rank]
        assert same and collage == int(g["collage_c2"])
        # the whole image's comparisons, from the gathered leaves == sum of the slabs'
        assert comps == res[0][3] + res[1][3]
    assert res[0][4] + res[1][4] == len(np.asarray(g["records_c2"]))


def _balanced_worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_1502_00324_b200 as fc
    from paper_1502_00324_b200 import _native

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = np.load(os.path.join(GOLDEN, "encode_c2.npz"))
    caps = tuple(int(v) for v in g["caps_c2"])
    params = fc.PoolParams(pool_cap=max(caps), strides=tuple(int(v) for v in g["strides_c2"]),
                           level_caps=caps)
    cfg = fc.EncoderConfig(pool=params, thresholds=tuple(float(v) for v in g["thresholds_c2"]))
    ctx = _native.Context(0)
    stream, report = fc.encode_balanced(fc.GrayImage(g["image_c2"]), cfg, context=ctx)
    q.put((rank, fc.serialize(stream) == g["bytes_c2"].tobytes(), int(report.collage_ssd),
           [ls["ranges"] for ls in report.level_stats]))
    dist.barrier()
    dist.destroy_process_group()


def test_encode_balanced_two_processes_c2_bytes():
    """Per-level re-balanced sharding: each level's ranges split evenly over 2
    ranks (gloo, both on cuda:0), results all-gathered; stream == golden."""
    g = np.load(os.path.join(GOLDEN, "encode_c2.npz"))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_balanced_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {r[0]: r[1:] for r in (q.get(timeout=600) for _ in procs)}
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank in (0, 1):
        same, collage, shares = res[rank]
        assert same and collage == int(g["collage_c2"])
    # every level's shares differ by at most one range
    for a, b in zip(res[0][2], res[1][2]):
        assert abs(a - b) <= 1


def _tau_worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_1502_00324_b200 as fc
    from paper_1502_00324_b200 import _native, workloads as W

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # entropy-threshold pools (c2's frozen p90 taus): the ranks' survivor
    # lists are all-gathered, then ranked on every rank
    img = fc.GrayImage(W.WORKLOADS["c2"].image(0))
    cfg = W.encoder_config("c2")
    ctx = _native.Context(0)
    stream, report = fc.encode_distributed(img, cfg, context=ctx)
    single, srep = fc.encode(img, cfg, context=_native.Context(0))
    q.put((rank, fc.serialize(stream) == fc.serialize(single), tuple(report.pool_sizes),
           tuple(srep.pool_sizes)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_encode_distributed_sharded_threshold_pool_matches_single_process(world):
    """world 3: window-row blocks of unequal fill (481 / 497 / 505 / 509 rows
    per level over 3 ranks) and survivor lists of different lengths."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tau_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r[0]: r[1:] for r in (q.get(timeout=600) for _ in procs)}
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank in range(world):
        same, sizes, single_sizes = res[rank]
        assert same and sizes == single_sizes


def _nccl_worker(port, q):
    import torch
    import torch.distributed as dist

    import paper_1502_00324_b200 as fc
    from paper_1502_00324_b200 import _native, workloads as W

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    out = []
    for name in ("c2", "c1"):  # threshold pools, then caps with cap-1 levels
        img = fc.GrayImage(W.WORKLOADS[name].image(0))
        cfg = W.encoder_config(name)
        a = fc.build_pool_sharded(img, cfg.pool, context=_native.Context(0), force=True)
        b = fc.build_pool(img, cfg.pool, context=_native.Context(0))
        same = a.sizes == b.sizes and all(
            np.array_equal(np.asarray(a.coords(lv)), np.asarray(b.coords(lv))) and
            np.array_equal(a.means(lv), b.means(lv)) for lv in (1, 2, 3, 4))
        out.append((name, bool(same)))
    q.put(out)
    dist.destroy_process_group()


def test_sharded_pool_exchange_over_nccl_single_rank():
    """The sharded pool build's exchange on the NCCL backend (device tensors,
    the context stream ordered around the collectives): one rank, forced
    through the exchange path, gives build_pool's pool."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    res = q.get(timeout=600)
    p.join(timeout=120)
    assert p.exitcode == 0
    assert all(same for _, same in res), res


def _c5_worker(rank, world, port, q):
    import hashlib

    import torch.distributed as dist

    import paper_1502_00324_b200 as fc
    from paper_1502_00324_b200 import _native, workloads as W

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    img = fc.GrayImage(W.WORKLOADS["c5"].image(0))
    cfg = W.encoder_config("c5")
    stream, report = fc.encode_distributed(img, cfg, context=_native.Context(0))
    digest = hashlib.sha256(fc.serialize(stream)).hexdigest()
    single = None
    if rank == 0:
        s1, _ = fc.encode(img, cfg, context=_native.Context(0))
        single = hashlib.sha256(fc.serialize(s1)).hexdigest()
    q.put((rank, digest, single, tuple(report.pool_sizes)))
    dist.barrier()
    dist.destroy_process_group()


def test_c5_encode_distributed_eight_processes_matches_single_process():
    """The bench's default workload as the 8-GPU scaling run partitions it
    (8 range slabs, the 4.13 M-window entropy pass sharded and all-gathered),
    here as 8 gloo processes on one GPU: every rank's stream equals the
    single-process encode's bytes."""
    world = 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_c5_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r[0]: r[1:] for r in (q.get(timeout=900) for _ in procs)}
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    single = res[0][1]
    assert single is not None
    for rank in range(world):
        assert res[rank][0] == single, rank
        assert res[rank][2] == (1, 4133089, 1, 1)
