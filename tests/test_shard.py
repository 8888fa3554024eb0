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
