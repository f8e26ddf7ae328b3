"""Host-side logic of the multi-GPU mode on CPU: the Morton partition (no device needed) and the
range all-gather under a 2-rank gloo group."""
import os
import socket

import numpy as np
import pytest

from paper_1803_09948_b200 import api
from paper_1803_09948_b200.workloads import plummer_points, sphere_points


@pytest.mark.parametrize("xyz,k,ncrit,cap,theta", [
    (sphere_points(20000, 1), 4.0, 64, 0.25, 0.4),
    (plummer_points(15000, 2, 0.05), 8.0, 64, 0.125, 0.35),
])
@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_morton_partition_tiles_and_balances(xyz, k, ncrit, cap, theta, nranks):
    tree = api.debug_host_tree(xyz, ncrit, cap, k, theta, 1.0)
    cells = tree["cells"]
    first, count, cell_rank, lcut = api.debug_partition(xyz, ncrit, cap, k, theta, 1.0, nranks, len(cells))
    # contiguous ranges that tile the Morton order in rank order
    assert first[0] == 0 and (first[1:] == (first + count)[:-1]).all() and first[-1] + count[-1] == len(xyz)
    lv = cells[:, 0].astype(int)
    # cells at or below the cut (and leaves above it) have exactly one owner, consistent with the
    # body range of that owner; cells above the cut hold no expansion and have none
    owned = cell_rank >= 0
    assert (owned == ((lv >= lcut) | (cells[:, 7] == 0))).all()
    r = cell_rank[owned]
    bf, bc = cells[owned, 4].astype(np.int64), cells[owned, 5].astype(np.int64)
    assert ((bf >= first[r]) & (bf + bc <= first[r].astype(np.int64) + count[r])).all()
    # children inherit their parent's owner
    for c in np.nonzero(owned & (cells[:, 7] > 0))[0][:500]:
        ch = slice(cells[c, 6], cells[c, 6] + cells[c, 7])
        assert (cell_rank[ch] == cell_rank[c]).all()
    # estimated work per rank (the partition's own weights) is balanced within the unit granularity
    m2l_t = tree["m2l"][:, 0]
    p2p = tree["p2p"]
    w = np.zeros(nranks)
    np.add.at(w, cell_rank[m2l_t], 1600.0)
    np.add.at(w, cell_rank[p2p[:, 0]], cells[p2p[:, 0], 5].astype(float) * cells[p2p[:, 1], 5])
    assert w.min() > 0
    assert w.max() / w.mean() < (1.6 if nranks <= 4 else 2.2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1803_09948_b200.distributed import allgather_ranges

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rows owned per rank: two ranges each (as two tree levels), uneven sizes
        ranges = [[(0, 3), (10, 2)], [(3, 7), (12, 5)]]
        truth = torch.arange(17 * 4, dtype=torch.float32).reshape(17, 4)
        buf = torch.full((17, 4), -1.0)
        for f, c in ranges[rank]:
            buf[f:f + c] = truth[f:f + c]
        scratch = allgather_ranges(dist, buf, ranges, rank, world)
        ok1 = bool((buf == truth).all())
        # reuse of the scratch buffers, 1-D payload, body-range style
        br = [[(0, 9)], [(9, 4)]]
        v = torch.zeros(13, 2)
        v[br[rank][0][0]:br[rank][0][0] + br[rank][0][1]] = float(rank + 1)
        allgather_ranges(dist, v, br, rank, world)
        ok2 = bool((v[:9] == 1).all() and (v[9:] == 2).all())
        # locally-essential-tree exchange: uneven all_to_all with index lists (rows sent to the peer /
        # rows received from it), in place
        from paper_1803_09948_b200.distributed import exchange_rows
        truth = torch.arange(12 * 3, dtype=torch.float32).reshape(12, 3)
        own = [torch.tensor([0, 1, 2, 3, 4, 5]), torch.tensor([6, 7, 8, 9, 10, 11])]
        need = [torch.tensor([7, 10, 11]), torch.tensor([1, 4])]      # rows rank r needs from the other rank
        buf = torch.full((12, 3), -1.0)
        buf[own[rank]] = truth[own[rank]]
        empty = torch.zeros(0, dtype=torch.int64)
        send = [empty, empty]
        recv = [empty, empty]
        send[1 - rank] = need[1 - rank]
        recv[1 - rank] = need[rank]
        exchange_rows(dist, buf, send, recv, "cpu")
        have = torch.cat([own[rank], need[rank]])
        rest = torch.tensor([i for i in range(12) if i not in set(have.tolist())])
        ok3 = bool((buf[have] == truth[have]).all() and (buf[rest] == -1).all())
        q.put((rank, ok1 and ok2 and ok3 and scratch is not None))
    finally:
        dist.destroy_process_group()


def test_range_allgather_two_ranks_gloo():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)]
