"""Request-level data parallelism across GPUs: one process per
GPU, each serving a contiguous shard of the request stream with a full
replica of the base model and caches. No collective touches the serve path;
torch.distributed (NCCL on GPUs, gloo in the CPU tests) is used only for the
barrier around the timed region, the max-over-ranks time and the final
request-ordered gather of the per-request traces.

The reference serves requests sequentially and independently
(serving.cpp:154-156 loops serve_one over the stream; serve_one reads only
const model state), so sharding is exact: the gathered traces equal a
single-process run.
"""
from __future__ import annotations

from typing import Callable, Dict, Tuple

import numpy as np


def shard_bounds(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) of n requests for `rank`; sizes differ by <= 1."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("shard_bounds: rank outside [0, world)")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (device time of the timed region)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_traces(local: Dict[str, np.ndarray], n_total: int, dist=None) -> Dict[str, np.ndarray]:
    """Concatenate per-rank result arrays (first axis = this rank's requests, in
    shard order) into request order on every rank."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return {k: np.asarray(v) for k, v in local.items()}
    world = dist.get_world_size()
    parts = [None] * world
    dist.all_gather_object(parts, {k: np.asarray(v) for k, v in local.items()})
    out = {k: np.concatenate([p[k] for p in parts], axis=0) for k in local}
    for k, v in out.items():
        if v.shape[0] != n_total:
            raise RuntimeError(f"gather_traces: {k} has {v.shape[0]} rows, expected {n_total}")
    return out


def serve_sharded(serve_fn: Callable[[np.ndarray], Dict[str, np.ndarray]], inputs: np.ndarray, dist=None
                  ) -> Dict[str, np.ndarray]:
    """Serve this rank's contiguous shard of `inputs` with `serve_fn` (a replica:
    Deployment.serve on this rank's GPU, or the CPU oracle in tests) and return
    the request-ordered traces of the whole stream."""
    world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    lo, hi = shard_bounds(inputs.shape[0], rank, world)
    local = serve_fn(inputs[lo:hi]) if hi > lo else None
    if local is None:
        probe = serve_fn(inputs[:1])
        local = {k: np.asarray(v)[:0] for k, v in probe.items()}
    return gather_traces(local, inputs.shape[0], dist)
