"""Request-level data parallelism: one process per GPU, each owning its requests' KV
pages and a full weight replica; no exchange on the data path.  torch.distributed (NCCL on GPUs,
gloo in the CPU tests) is used only to aggregate timing / decode statistics and to gather outputs."""
from __future__ import annotations

import os
from typing import Sequence


def env_world():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def init(backend: str = "nccl"):
    """Initialise the default process group when launched under torchrun (WORLD_SIZE > 1)."""
    import torch.distributed as dist
    rank, world, local = env_world()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return rank, world, local


def shard_requests(n_total: int, world: int, rank: int, costs: Sequence[float] | None = None) -> list:
    """Global request ids owned by `rank`.  Equal counts per rank; with costs (e.g. prompt length +
    gen/2, the attention bytes a request streams per step) requests are dealt longest-first to the
    least-loaded rank that still has room (LPT with equal counts)."""
    if costs is None:
        per = n_total // world
        extra = n_total % world
        lo = rank * per + min(rank, extra)
        return list(range(lo, lo + per + (1 if rank < extra else 0)))
    cap = [n_total // world + (1 if r < n_total % world else 0) for r in range(world)]
    load = [0.0] * world
    owner = {}
    for i in sorted(range(n_total), key=lambda i: (-costs[i], i)):
        r = min((r for r in range(world) if cap[r] > 0), key=lambda r: (load[r], r))
        owner[i] = r
        load[r] += costs[i]
        cap[r] -= 1
    return sorted(i for i in range(n_total) if owner[i] == rank)


def reduce_max(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_min(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return float(t.item())


def reduce_sum(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def all_gather_stats(stats: Sequence[int], device=None) -> list:
    """All-gather a small int64 vector of per-rank statistics -> list of per-rank lists."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return [list(stats)]
    t = torch.tensor(list(stats), dtype=torch.int64, device=device)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.tolist() for o in out]


def gather_outputs(local: dict, device=None) -> dict:
    """Gather {global request id: committed token ids} from every rank (all ranks receive the union).
    Requests are independent, so the union is identical for any world size."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return dict(local)
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, {int(k): list(map(int, v)) for k, v in local.items()})
    out = {}
    for p in parts:
        for k, v in p.items():
            assert k not in out, f"request {k} owned by two ranks"
            out[k] = v
    return out


def barrier(device=None):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        if device is not None and dist.get_backend() == "nccl":
            dist.barrier(device_ids=[device.index if hasattr(device, "index") else int(device)])
        else:
            dist.barrier()
