"""N > 1 host logic of `bench.py --gpus N` on CPU (world_size 2, gloo):
per-rank seeding, max-over-ranks timing and the whole-job rate
(paper_2506_17626_b200/replicas.py)."""

import json
import os
import socket

import numpy as np
import pytest


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir):
    import torch.distributed as dist
    from paper_2506_17626_b200 import workloads
    from paper_2506_17626_b200.replicas import (barrier, max_over_ranks, replica_seed,
                                                 whole_job_rate)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        elapsed = max_over_ranks(1.5 + rank)
        barrier()
        wl = workloads.build("cfg1", seed=replica_seed(rank))
        digests = [None] * world
        dist.all_gather_object(digests, float(np.asarray(wl.basis.weights[0]).sum()))
        res = dict(rank=rank, elapsed=elapsed, rate=whole_job_rate(world, 3, elapsed),
                   digests=digests)
        with open(os.path.join(outdir, f"r{rank}.json"), "w") as fh:
            json.dump(res, fh)
    finally:
        dist.destroy_process_group()


def test_two_replicas_gloo(tmp_path):
    mp = pytest.importorskip("torch.multiprocessing")
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    out = [json.load(open(tmp_path / f"r{r}.json")) for r in range(world)]
    for r in out:
        assert r["elapsed"] == 2.5                     # max over ranks, on every rank
        assert r["rate"] == pytest.approx(world * 3 / 2.5)
        assert r["digests"] == out[0]["digests"]
    d = out[0]["digests"]
    assert d[0] != d[1]                                # each replica solves its own seed


def test_single_process_helpers():
    from paper_2506_17626_b200.replicas import max_over_ranks, replica_seed, whole_job_rate
    assert max_over_ranks(3.25) == 3.25
    assert replica_seed(5) == 5
    assert whole_job_rate(1, 2, 4.0) == 0.5
