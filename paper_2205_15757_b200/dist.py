"""Multi-GPU plumbing: one process per GPU over torch.distributed.

* :func:`assigned_models` — the reference's deterministic model partition
  (proj/src/domain.cpp:247-268): which models of a group node ``rank`` serves.
  With one replica per GPU (|G| == N) it is the bijection rank -> model.
* :func:`share_bytes` — broadcast rank 0's NCCL unique id (or any bytes).
* :func:`max_over_ranks` — the timing rule: max of a per-rank duration.

The data path's collective (the all-gather of replica outputs and R roots)
is NCCL inside libcredo_gpu.so (cg_group_create_dist); torch.distributed only
rendezvouses and times.
"""
from __future__ import annotations

import os


def assigned_models(owner_node_count: int, n_models: int, node_index: int) -> list[int]:
    """Indices of the group's models that node ``node_index`` serves.

    domain.cpp:247-268: the ordered model list is split into contiguous
    chunks of ceil(|G|/d) models; node k serves chunk (k mod num_chunks)."""
    if owner_node_count < 1:
        raise ValueError("assigned_models: no owner nodes")
    if n_models < 1:
        raise ValueError("assigned_models: empty group")
    if node_index >= owner_node_count:
        raise ValueError("assigned_models: node rank out of range")
    g, d = n_models, owner_node_count
    chunk_size = (g + d - 1) // d
    num_chunks = (g + chunk_size - 1) // chunk_size
    chunk = node_index % num_chunks
    begin = chunk * chunk_size
    return list(range(begin, min(begin + chunk_size, g)))


def env_rank() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def share_bytes(data: bytes | None) -> bytes:
    """Rank 0's bytes on every rank (object broadcast; gloo or nccl)."""
    import torch.distributed as dist
    obj = [data]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
