"""Host logic of the multi-GPU path: the target-range
partition (C ABI, host only) and the torch.distributed bootstrap, with
world_size-2 gloo process groups on CPU."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from hypothesis import given, settings, strategies as st


@pytest.fixture(scope="module")
def P():
    from paper_2107_04092_b200 import build_ext
    build_ext.build()
    import paper_2107_04092_b200 as P
    return P


@settings(max_examples=200, deadline=None)
@given(st.integers(0, 3_000_000), st.sampled_from([32, 64, 256, 1024, 4096]), st.integers(1, 8))
def test_partition_tiles_target_range(n, C, world):
    from paper_2107_04092_b200.dist import partitions
    parts = partitions(n, C, world)
    assert parts[0][0] == 0 and parts[-1][1] == n
    for (lo, hi), (lo2, _) in zip(parts, parts[1:]):
        assert hi == lo2                          # contiguous, disjoint
    for lo, hi in parts:
        assert lo <= hi
        if lo < n:
            assert lo % C == 0                    # slices never straddle ranks
            assert lo % 32 == 0                   # nor do spike-bitmask words
    sizes = [hi - lo for lo, hi in parts]
    share = sizes[0]
    assert all(s <= share for s in sizes)         # equal shares, the tail truncated


@settings(max_examples=200, deadline=None)
@given(st.lists(st.floats(0.0, 1e3), min_size=1, max_size=300), st.sampled_from([32, 96, 1024]),
       st.integers(1, 8), st.integers(0, 31))
def test_weighted_partition_tiles_and_balances(cost, C, world, tail):
    from paper_2107_04092_b200.snn import snn_partition_weighted
    n = max(0, len(cost) * C - tail)
    parts = [snn_partition_weighted(cost, n, C, world, r) for r in range(world)]
    assert parts[0][0] == 0 and parts[-1][1] == n
    for (lo, hi), (lo2, _) in zip(parts, parts[1:]):
        assert hi == lo2 and lo <= hi
    for lo, _ in parts:
        assert lo % C == 0 or lo == n                  # slices never straddle ranks
    # each rank's cost is within one slice of the ideal share (boundaries are
    # the slice prefixes closest to r / world of the total)
    total, cmax = sum(cost), max(cost)
    for lo, hi in parts:
        got = sum(cost[lo // C:(hi + C - 1) // C]) if hi > lo else 0.0
        assert abs(got - total / world) <= 2 * cmax + 1e-9 * total


def test_weighted_partition_spreads_plastic_targets():
    """BASELINE config 4 layout: E (plastic targets, costlier) then I; with
    world 8 the E range is split over more ranks than an equal neuron split."""
    from paper_2107_04092_b200.snn import snn_partition_weighted
    C, nE, nI = 512, 252_982, 63_246
    R = nE + nI
    ns = (R + C - 1) // C
    cost = []
    for k in range(ns):
        a, b = k * C, min(R, (k + 1) * C)
        e = max(0, min(b, nE) - a)
        cost.append(e * 9.0 + (b - a - e) * 1.0)
    parts = [snn_partition_weighted(cost, R, C, 8, r) for r in range(8)]
    n_e_ranks = sum(1 for lo, hi in parts if lo < nE)
    assert n_e_ranks == 8                               # every rank gets plastic targets
    shares = [sum(cost[lo // C:(hi + C - 1) // C]) for lo, hi in parts]
    assert max(shares) / min(shares) < 1.05


def test_partition_rejects_bad_arguments(P):
    for args in [(100, 1000, 2, 0), (100, 1024, 0, 0), (100, 1024, 2, 2)]:
        with pytest.raises(P.SnnError):
            P.snn_partition(*args)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2107_04092_b200 as P
        from paper_2107_04092_b200 import dist as pd
        # every rank derives its own range; gathered, they must tile [0, R)
        R, C = 158_114, 1024
        mine = P.snn_partition(R, C, world, rank)
        allr = [None] * world
        dist.all_gather_object(allr, mine)
        # the bootstrap of the communicator: one id, broadcast from rank 0
        torch.cuda.nccl.unique_id = lambda: os.urandom(128)   # no GPU here: stand-in id
        uid = pd.nccl_unique_id()
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        q.put((rank, allr, len(set(ids)), len(uid)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_partition_and_id_broadcast(P):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, allr, n_ids, ln in res:
        assert allr == [tuple(x) for x in P.dist.partitions(158_114, 1024, world)]
        assert n_ids == 1 and ln == 128
