"""World-size-2 CPU (gloo) tests of the multi-rank host logic: every rank derives its own
contiguous output range from (D, world, rank) alone (no data-path collective), the ranges
tile [0, 3^D) exactly, and bench.py's max-over-ranks timing reduction picks the slowest rank."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, D, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1608_00206_b200.hc as hc
        import bench
        b, e = hc.shard_range(D, world, rank)
        mine = torch.tensor([b, e], dtype=torch.int64)
        allr = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allr, mine)
        # bench's timing reduction: each rank reports (elapsed_ms, kernel_ms); max over ranks
        t = bench.reduce_max([10.0 + rank, 3.0 * (world - rank)], dist, device="cpu")
        q.put((rank, [tuple(int(v) for v in r) for r in allr], t))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("D", [16, 20, 22])
def test_two_rank_partition_and_timing(D):
    import paper_1608_00206_b200.build as b
    b.build()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, D, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    ranges = res[0][1]
    assert all(r[1] == ranges for r in res)          # every rank sees the same split
    assert ranges[0][0] == 0 and ranges[-1][1] == 3 ** D
    assert ranges[0][1] == ranges[1][0]
    for _, _, t in res:
        assert t == [10.0 + world - 1, 3.0 * world]   # max over ranks, elementwise


def _ep_worker(rank, world, port, D, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1608_00206_b200.hc as hc
        (e0, e1), (c0, c1) = hc.ep_range(D, k, world, rank)
        nc = 3 ** (D - k)
        # w rows of this rank's points, value = e * 10^6 + column (exact in float64)
        e = torch.arange(e0, e1, dtype=torch.float64).view(-1, 1)
        w = (e * 1e6 + torch.arange(nc, dtype=torch.float64).view(1, -1)).reshape(-1)
        wt = torch.full(((3 ** k) * (c1 - c0),), -1.0, dtype=torch.float64)
        hc.ep_exchange(w, wt, D, k, rank, world, dist)
        want = (torch.arange(3 ** k, dtype=torch.float64).view(-1, 1) * 1e6
                + torch.arange(c0, c1, dtype=torch.float64).view(1, -1)).reshape(-1)
        q.put((rank, bool(torch.equal(wt, want))))
    except Exception as ex:  # report instead of leaving the parent waiting on the queue
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("D,k", [(8, 2), (9, 3), (10, 5)])
def test_two_rank_evalpoint_exchange(D, k):
    # the all-to-all of the evaluation-point variant (north_star (4)): after the exchange each
    # rank holds every point's values on exactly its own columns
    import paper_1608_00206_b200.build as b
    b.build()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ep_worker, args=(r, world, port, D, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok is True for _, ok in res), res
