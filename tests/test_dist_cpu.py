"""CPU, world_size 2 over gloo: the host-side multi-GPU logic (rendezvous on
127.0.0.1, NCCL-id broadcast, max-over-ranks timing) and the reference's
replica<->node partition (proj/src/domain.cpp:247-268, properties pinned by
tests/test_domain.cpp:90-151)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2205_15757_b200.dist import assigned_models


def test_assigned_models_properties():
    # test_domain.cpp:135-151: every node nonempty, cover, over [1,8]^2
    for d in range(1, 9):
        for g in range(1, 9):
            sets = [assigned_models(d, g, k) for k in range(d)]
            assert all(len(s) >= 1 for s in sets)
            assert set().union(*map(set, sets)) == set(range(g))
    # :90-102 bijection when |G| = d
    assert [assigned_models(4, 4, k) for k in range(4)] == [[0], [1], [2], [3]]
    # :104-118 disjoint cover when |G| > d
    assert [assigned_models(2, 4, k) for k in range(2)] == [[0, 1], [2, 3]]
    # :120-133 replication when |G| < d: each model held by two nodes
    holders = [assigned_models(4, 2, k) for k in range(4)]
    assert all(len(h) == 1 for h in holders)
    assert sorted(h[0] for h in holders) == [0, 0, 1, 1]
    # :153-158 and the range checks (domain.cpp:250-258)
    for args in [(4, 0, 0), (0, 4, 0), (4, 4, 4)]:
        with pytest.raises(ValueError):
            assigned_models(*args)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2205_15757_b200.dist import max_over_ranks, share_bytes
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = share_bytes(bytes(range(128)) if rank == 0 else None)
    m = max_over_ranks(10.0 + rank)
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, uid == bytes(range(128)), m))


def test_two_rank_gloo_rendezvous():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == [(0, True, 11.0), (1, True, 11.0)]
