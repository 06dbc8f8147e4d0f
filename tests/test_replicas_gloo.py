"""The N>1 (replicas-only) path on CPU: world_size 2 over gloo, exercising the
same barrier / max-over-ranks / throughput code bench.py uses with nccl."""
import os
import socket

import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    from paper_2009_00083_b200 import replicas as R
    r, w, lr = R.init("gloo")
    assert (r, w, lr) == (rank, world, rank)
    R.barrier()
    per_rank_ms = 10.0 + 5.0 * rank  # rank 1 is the slowest
    m = R.max_over_ranks(per_rank_ms)
    out[rank] = m
    out[world + rank] = R.job_throughput(1000, w, m)
    R.shutdown()


def test_replicas_gloo_world2():
    world = 2
    out = torch.zeros(2 * world, dtype=torch.float64).share_memory_()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0].item() == out[1].item() == 15.0
    # 2 ranks x 1000 units in 15 ms (slowest rank)
    assert abs(out[2].item() - 2 * 1000 / 0.015) < 1e-6


def test_single_process_defaults(monkeypatch):
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        monkeypatch.delenv(k, raising=False)
    from paper_2009_00083_b200 import replicas as R
    assert R.env() == (0, 1, 0)
    assert R.max_over_ranks(3.5) == 3.5
    assert R.job_throughput(100, 1, 10.0) == 10000.0
