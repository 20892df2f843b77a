"""Replica-parallel certification over NCCL (one process per GPU, rank =
provider; cg_group_create_dist). Every rank must produce the same
certificate as a single-GPU group holding all N replicas — and, with three
ranks, the reference's own golden certificate (tests/golden/c1_batch.npz).

Needs >= 2 GPUs (`gpurun --gpus 2|4`); skipped on a 1-GPU box."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT, golden, split_reqs

pytestmark = pytest.mark.gpu

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
KEYS = ("selected", "diameter", "satisfied", "label", "r_roots", "a_root",
        "manifest_len", "manifest_kind", "manifest_node", "manifest_op", "a_leaf_hashes")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, f, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from paper_2205_15757_b200 import EUCLIDEAN, Context, Model, ModelGroup, RequestBatch
    from paper_2205_15757_b200.dist import assigned_models, share_bytes
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        g = golden("c1_batch.npz")
        B = int(g["B"])
        ctx = Context(rank)
        uid = share_bytes(Context.nccl_unique_id() if rank == 0 else None)
        ctx.init_nccl(uid, world, rank)
        mine = assigned_models(world, N, rank)  # |G| == d: the bijection; else chunks
        ms = [Model.load_linear(ctx, g["files"][p % 3].tobytes(), g["digests"][p % 3].tobytes())
              for p in mine]
        digests = [g["digests"][i % 3].tobytes() for i in range(N)]
        grp = ModelGroup.create_dist(ctx, ms if len(ms) > 1 else ms[0], digests, f, EUCLIDEAN,
                                     float(g["eps"]), g["gid"].tobytes(), 1, max_batch=B, topk=3)
        batch = RequestBatch.from_encoded(split_reqs(g))
        r1 = grp.certify(batch, want_outputs=True)
        # pipelined path: ingest ahead, certify later
        t0, t1 = grp.ingest(batch), grp.ingest(batch)
        grp.certify_ticket(t0)
        r2 = grp.certify_ticket(t1)
        r3 = grp.certify_outputs(batch, g["partial_fault_outputs"][[i % 3 for i in range(N)]])
        out = {k: (r1[k], r2[k], r3[k]) for k in KEYS}
        out["outputs"] = r1["outputs"]
        grp.free()
        for m in ms:
            m.free()
        ctx.close()
        dist.destroy_process_group()
        q.put((rank, out, None))
    except Exception as e:  # surfaced in the parent
        q.put((rank, None, repr(e)))


def _run(world, N, f):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, N, f, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in ps:
        rank, out, err = q.get(timeout=600)
        assert err is None, f"rank {rank}: {err}"
        res[rank] = out
    for p in ps:
        p.join(timeout=120)
    return res


def _single(N, f):
    from paper_2205_15757_b200 import EUCLIDEAN, Context, Model, ModelGroup, RequestBatch
    g = golden("c1_batch.npz")
    B = int(g["B"])
    ctx = Context(0)
    ms = [Model.load_linear(ctx, g["files"][p % 3].tobytes(), g["digests"][p % 3].tobytes())
          for p in range(N)]
    grp = ModelGroup(ctx, ms, f, EUCLIDEAN, float(g["eps"]), g["gid"].tobytes(), 1,
                     max_batch=B, topk=3)
    batch = RequestBatch.from_encoded(split_reqs(g))
    r1 = grp.certify(batch, want_outputs=True)
    r3 = grp.certify_outputs(batch, g["partial_fault_outputs"][[i % 3 for i in range(N)]])
    out = {k: (r1[k], r3[k]) for k in KEYS}
    out["outputs"] = r1["outputs"]
    grp.free()
    for m in ms:
        m.free()
    ctx.close()
    return out


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_dist_two_ranks_equals_single_gpu_group():
    N, f = 2, 0
    res = _run(2, N, f)
    want = _single(N, f)
    for rank, out in res.items():
        assert np.array_equal(out["outputs"], want["outputs"]), rank
        for k in KEYS:
            r1, r2, r3 = out[k]
            assert np.array_equal(r1, want[k][0]), (rank, k)
            assert np.array_equal(r2, want[k][0]), (rank, k, "pipelined")
            assert np.array_equal(r3, want[k][1]), (rank, k, "outputs")


@pytest.mark.skipif(NGPU < 3, reason="needs >= 3 GPUs")
def test_dist_three_ranks_reference_golden():
    g = golden("c1_batch.npz")
    res = _run(3, 3, 1)
    for rank, out in res.items():
        assert np.array_equal(out["outputs"], g["outputs"]), rank
        r1, r2, _ = out["a_root"]
        assert r1.tobytes() == g["honest_a_root"].tobytes(), rank
        assert r2.tobytes() == g["honest_a_root"].tobytes(), rank
        assert np.array_equal(out["r_roots"][0], g["honest_r_roots"]), rank
        assert np.array_equal(out["selected"][0], g["honest_sel"].astype(np.uint32)), rank
        assert np.array_equal(out["label"][0], g["honest_label"]), rank
        assert np.array_equal(out["r_roots"][2], g["partial_fault_r_roots"]), rank
        assert out["a_root"][2].tobytes() == g["partial_fault_a_root"].tobytes(), rank


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_dist_two_replicas_per_rank_equals_single_gpu_group():
    """assigned_models chunking with |G| > d (domain.cpp:247-268): 4 providers
    on 2 ranks, 2 local replicas per rank (cg_group_create_dist_multi), one
    all-gather of 2 providers' outputs and R roots per rank."""
    N, f = 4, 1
    res = _run(2, N, f)
    want = _single(N, f)
    for rank, out in res.items():
        assert np.array_equal(out["outputs"], want["outputs"]), rank
        for k in KEYS:
            r1, r2, r3 = out[k]
            assert np.array_equal(r1, want[k][0]), (rank, k)
            assert np.array_equal(r2, want[k][0]), (rank, k, "pipelined")
            assert np.array_equal(r3, want[k][1]), (rank, k, "outputs")
