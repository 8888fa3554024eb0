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


# ---------------------------------------------------------------- adaptation
# Online adaptation (§8f rank 3) across request-sharded replicas. The
# reference's run_adaptation (serving.cpp:213-340) is one sequential loop:
# every retrain is staged as `pending` and lands (`live = *pending`,
# serving.cpp:303-315) at the first request with time >= swap_time, so the
# caches serving a request at time t are those of the last swap landed at a
# time <= t. A fleet keeps that rule: one trainer replica runs the reference
# loop (Deployment + lc_run_adaptation, GPU retraining), each landed swap is
# captured by the engine's swap hook and broadcast to every replica (NCCL on
# GPUs, gloo on CPU; off the serve path), and every replica applies swap k
# before the first request of its shard at time >= t_k. The gathered traces
# equal the single-process run.

from dataclasses import dataclass, field  # noqa: E402
from typing import List, Optional, Sequence  # noqa: E402


@dataclass
class VariantSwap:
    """One landed retrain: requests at time >= time_min are served by these
    caches (one serialized variant per attached cache, probe order)."""
    time_min: float
    blobs: List[bytes] = field(default_factory=list)


def _world(dist):
    if dist is None or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(), dist.get_rank()


def broadcast_bytes(blob: Optional[bytes], src: int = 0, dist=None, device=None) -> bytes:
    """rank `src`'s bytes on every rank (length, then payload; uint8 tensors on
    `device`: a CUDA device for NCCL, None/CPU for gloo)."""
    world, rank = _world(dist)
    if world == 1:
        if blob is None:
            raise ValueError("broadcast_bytes: the source rank must provide the payload")
        return bytes(blob)
    import torch
    n = torch.tensor([len(blob) if rank == src else 0], dtype=torch.int64, device=device)
    dist.broadcast(n, src)
    buf = torch.empty(int(n.item()), dtype=torch.uint8, device=device)
    if rank == src and len(blob):
        buf.copy_(torch.frombuffer(bytearray(blob), dtype=torch.uint8))
    dist.broadcast(buf, src)
    return bytes(buf.cpu().numpy().tobytes())


def pack_swaps(swaps: Sequence[VariantSwap]) -> bytes:
    """[u32 count] then per swap [f64 time][u32 n] + n x ([u64 len][bytes])."""
    import struct
    out = [struct.pack("<I", len(swaps))]
    for s in swaps:
        out.append(struct.pack("<dI", float(s.time_min), len(s.blobs)))
        for b in s.blobs:
            out.append(struct.pack("<Q", len(b)))
            out.append(bytes(b))
    return b"".join(out)


def unpack_swaps(data: bytes) -> List[VariantSwap]:
    import struct
    off = 0

    def take(fmt):
        nonlocal off
        v = struct.unpack_from(fmt, data, off)
        off += struct.calcsize(fmt)
        return v

    (count,) = take("<I")
    swaps = []
    for _ in range(count):
        t, n = take("<dI")
        blobs = []
        for _ in range(n):
            (ln,) = take("<Q")
            if off + ln > len(data):
                raise ValueError("unpack_swaps: truncated payload")
            blobs.append(bytes(data[off:off + ln]))
            off += ln
        swaps.append(VariantSwap(t, blobs))
    if off != len(data):
        raise ValueError("unpack_swaps: trailing bytes")
    return swaps


def broadcast_swaps(swaps: Optional[Sequence[VariantSwap]], src: int = 0, dist=None, device=None
                    ) -> List[VariantSwap]:
    """The trainer's landed swaps on every replica (one collective pair)."""
    _, rank = _world(dist)
    payload = pack_swaps(swaps) if rank == src else None
    return unpack_swaps(broadcast_bytes(payload, src, dist, device))


def swap_segments(times: Sequence[float], swaps: Sequence[VariantSwap]):
    """Contiguous [lo, hi) ranges of a time-ordered request list and the swap
    in effect for each (-1 = the initial caches): swap k covers requests with
    time >= swaps[k].time_min (serving.cpp:303-315)."""
    t = np.asarray(times, np.float64)
    if t.size > 1 and np.any(np.diff(t) < 0):
        raise ValueError("swap_segments: requests must be in time order")
    st = [s.time_min for s in swaps]
    if any(b < a for a, b in zip(st, st[1:])):
        raise ValueError("swap_segments: swaps must be in time order")
    segs, lo, k = [], 0, -1
    for j, ts in enumerate(st):
        hi = int(np.searchsorted(t, ts, side="left"))  # first request at time >= ts
        if hi > lo:
            segs.append((lo, hi, k))
            lo = hi
        k = j
    if t.size > lo:
        segs.append((lo, int(t.size), k))
    return segs


def serve_with_swaps(serve_fn: Callable[[np.ndarray], Dict[str, np.ndarray]], apply_fn: Callable[[VariantSwap], None],
                     inputs: np.ndarray, times: Sequence[float], swaps: Sequence[VariantSwap]
                     ) -> Dict[str, np.ndarray]:
    """One replica: serve time-ordered requests in segments, applying each swap
    (apply_fn) before the first request it covers. Swaps landing before the
    first request are applied up front, in order."""
    segs = swap_segments(times, swaps)
    applied = -1
    parts: List[Dict[str, np.ndarray]] = []
    for lo, hi, k in segs:
        while applied < k:
            applied += 1
            apply_fn(swaps[applied])
        parts.append({kk: np.asarray(v) for kk, v in serve_fn(inputs[lo:hi]).items()})
    while applied < len(swaps) - 1:  # swaps after the last request: the replica still ends on the final caches
        applied += 1
        apply_fn(swaps[applied])
    if not parts:
        probe = serve_fn(inputs[:1])
        return {k: np.asarray(v)[:0] for k, v in probe.items()}
    return {k: np.concatenate([p[k] for p in parts], axis=0) for k in parts[0]}


def serve_sharded_with_swaps(serve_fn, apply_fn, inputs: np.ndarray, times: Sequence[float],
                             swaps: Optional[Sequence[VariantSwap]], src: int = 0, dist=None, device=None
                             ) -> Dict[str, np.ndarray]:
    """Fleet serving under online adaptation: the trainer rank `src` provides
    the landed swaps, they are broadcast, every rank serves its contiguous
    shard of the time-ordered stream applying them, and the request-ordered
    traces are gathered on every rank."""
    world, rank = _world(dist)
    swaps = broadcast_swaps(swaps, src, dist, device)
    lo, hi = shard_bounds(inputs.shape[0], rank, world)
    local = serve_with_swaps(serve_fn, apply_fn, inputs[lo:hi], list(times)[lo:hi], swaps)
    return gather_traces(local, inputs.shape[0], dist)


def capture_swaps(dep) -> List[VariantSwap]:
    """Install a swap hook on a Deployment that records every swap
    run_adaptation lands (binary variants, probe order); returns the live list."""
    swaps: List[VariantSwap] = []

    def on_swap(t: float) -> None:
        swaps.append(VariantSwap(t, [dep.variant(k).save_binary() for k in range(len(dep.variants))]))

    dep.set_swap_hook(on_swap)
    return swaps


def apply_swap_to_deployment(dep, swap: VariantSwap) -> None:
    """Replica side of a swap: every cache's retrained networks into the engine
    (Deployment.update_variant, stream-ordered after the enqueued batches)."""
    from .api import load_variant_binary
    for b in swap.blobs:
        dep.update_variant(load_variant_binary(b))
