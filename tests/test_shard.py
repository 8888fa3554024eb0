"""Multi-GPU host logic on CPU: world_size-2 gloo processes shard the
reference's own golden request stream (tests/golden/trained, 3,600 traces
from the compiled reference pipeline), each rank serves its contiguous shard
with a replica (the CPU oracle stands in for the per-GPU engine here), and
the request-ordered gather equals the reference traces exactly. Also checks
shard bounds and the max-over-ranks reduction used for bench timing."""
import os
import socket
import sys

import numpy as np
import pytest

from tests.helpers import GOLDEN, ROOT

from paper_2101_07344_b200.shard import shard_bounds


def test_shard_bounds_partition():
    for n in (0, 1, 7, 256, 1001):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, _) in zip(spans, spans[1:]):
                assert b == c and b >= a
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2101_07344_b200.shard import max_over_ranks, serve_sharded
    from tests.test_oracle import _trained

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model, caches, X, reqs, traces = _trained()
    idx = [s for _, s in reqs]
    inputs = X[idx]

    def serve(xs):
        el, sv, bp, _ = O.oracle_serve_mlp(model, caches, xs)
        return {"exit_layer": el, "served": sv, "base_pred": bp}

    res = serve_sharded(serve, inputs, dist)
    t = max_over_ranks(1.5 + rank, dist)
    if rank == 0:
        np.savez(out_path, t=t, **res)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_serve_matches_reference_traces(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r = np.load(out)
    traces = [l.split() for l in open(os.path.join(GOLDEN, "trained", "traces.txt")).read().split("\n")[1:]
              if l and not l.startswith("#")]
    assert r["t"] == 2.5  # max over ranks
    assert r["exit_layer"].tolist() == [int(t[5]) for t in traces]
    assert r["served"].tolist() == [int(t[4]) for t in traces]
    assert r["base_pred"].tolist() == [int(t[3]) for t in traces]


# ------------------------------------------------------- adaptation swaps
def test_swap_segments_follow_the_reference_swap_rule():
    """serving.cpp:303-315: a landed swap serves every request at time >= its
    swap time; two swaps landing before the same request both apply, in order."""
    from paper_2101_07344_b200.shard import VariantSwap, swap_segments
    t = [0.0, 1.0, 1.5, 2.0, 4.0, 4.0, 7.5]
    sw = [VariantSwap(1.5), VariantSwap(1.5), VariantSwap(4.0), VariantSwap(9.0)]
    assert swap_segments(t, sw) == [(0, 2, -1), (2, 4, 1), (4, 7, 2)]
    assert swap_segments(t, []) == [(0, 7, -1)]
    assert swap_segments([], sw) == []
    with pytest.raises(ValueError):
        swap_segments([1.0, 0.5], sw)


def test_pack_swaps_round_trip():
    from paper_2101_07344_b200.shard import VariantSwap, pack_swaps, unpack_swaps
    sw = [VariantSwap(0.25, [b"abc", b""]), VariantSwap(15.0, [bytes(range(256)) * 3])]
    back = unpack_swaps(pack_swaps(sw))
    assert [(s.time_min, s.blobs) for s in back] == [(s.time_min, s.blobs) for s in sw]
    with pytest.raises(ValueError):
        unpack_swaps(pack_swaps(sw)[:-1])


def _golden_swaps():
    """Two retrain swaps mid-stream: the golden trained caches with other
    thresholds (binary variants, probe order), as a trainer would broadcast."""
    import paper_2101_07344_b200 as lcb
    from paper_2101_07344_b200.shard import VariantSwap
    d = os.path.join(GOLDEN, "trained")
    texts = []
    k = 0
    while os.path.exists(os.path.join(d, f"variant_{k}.txt")):
        texts.append(open(os.path.join(d, f"variant_{k}.txt")).read())
        k += 1
    swaps = []
    # layer-1 cache never fires (all exit at layer 2), then neither the first nor the second
    for t, deltas in ((12.0, (1.5, 0.0)), (25.0, (1.5, 1.5))):
        blobs = []
        for txt, dl in zip(texts, deltas):
            v = lcb.load_variant(txt)
            v.delta = dl
            blobs.append(v.save_binary())
        swaps.append(VariantSwap(t, blobs))
    return swaps


def _oracle_replica(model, caches):
    """A CPU replica: the oracle serve over the live caches; swaps replace them."""
    import paper_2101_07344_b200 as lcb
    from oracle import oracle as O
    live = {c[0]: c for c in caches}

    def apply(swap):
        for b in swap.blobs:
            v = lcb.load_variant_binary(b)
            pred, sel, d = O.variant_layers_from_product(v)
            live[v.layer] = (v.layer, pred, sel, d)

    def serve(xs):
        el, sv, bp, _ = O.oracle_serve_mlp(model, [live[l] for l in sorted(live)], xs)
        return {"exit_layer": el, "served": sv, "base_pred": bp}

    return serve, apply


def _fleet_worker(rank, world, port, out_path):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2101_07344_b200.shard import serve_sharded_with_swaps, serve_with_swaps
    from tests.test_oracle import _trained

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model, caches, X, reqs, traces = _trained()
    inputs = X[[s for _, s in reqs]]
    times = [float(t[1]) for t in traces]
    swaps = _golden_swaps() if rank == 0 else None  # only the trainer holds them
    serve, apply = _oracle_replica(model, caches)
    res = serve_sharded_with_swaps(serve, apply, inputs, times, swaps, src=0, dist=dist)
    if rank == 0:
        s1, a1 = _oracle_replica(model, caches)
        single = serve_with_swaps(s1, a1, inputs, times, swaps)
        s0, _ = _oracle_replica(model, caches)
        frozen = s0(inputs)
        np.savez(out_path, **{f"fleet_{k}": v for k, v in res.items()},
                 **{f"single_{k}": v for k, v in single.items()}, **{f"frozen_{k}": v for k, v in frozen.items()})
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_swap_broadcast_matches_single_replica(tmp_path):
    """Only rank 0 (the trainer) holds the swaps; after the broadcast every
    rank serves its shard applying them by the reference rule, and the
    gathered traces equal one replica serving the whole stream with the same
    swaps (and differ from the frozen caches: the swaps matter)."""
    import torch.multiprocessing as mp
    out = str(tmp_path / "fleet.npz")
    mp.spawn(_fleet_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r = np.load(out)
    for k in ("exit_layer", "served", "base_pred"):
        assert np.array_equal(r[f"fleet_{k}"], r[f"single_{k}"]), k
    assert not np.array_equal(r["fleet_exit_layer"], r["frozen_exit_layer"])
    assert np.array_equal(r["fleet_base_pred"], r["frozen_base_pred"])  # swaps touch the caches only
