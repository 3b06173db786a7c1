"""Multi-process host logic of bench.py on CPU (gloo, world size 2): max-over-ranks timing,
whole-job aggregation and sample sharding.  No GPU involved."""
import os
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    import benchlib
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ms = [12.5, 20.0][rank]
    m = benchlib.max_over_ranks(ms, dist)
    lo, hi = benchlib.shard(8, rank, world)
    out[rank] = (m, benchlib.aggregate(30, world, m), lo, hi)
    dist.destroy_process_group()


def test_two_rank_timing_and_sharding():
    import random
    port = 29500 + random.randint(0, 2000)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0][0] == out[1][0] == 20.0                    # max over ranks, seen by both
    assert abs(out[0][1] - 30 * 2 / 0.020) < 1e-9           # whole-job iterations / max time
    assert (out[0][2], out[0][3], out[1][2], out[1][3]) == (0, 4, 4, 8)


def test_shard_covers_all_units():
    sys.path.insert(0, ROOT)
    import benchlib
    for n in (1, 7, 8, 9):
        for w in (1, 2, 3, 8):
            spans = [benchlib.shard(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
