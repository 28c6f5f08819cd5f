"""World-size-2 checks of the replicas-only multi-GPU host logic on CPU with the
gloo backend: distinct per-rank batches and the max-over-ranks / sum-over-ranks reduction that
bench.py applies to the timed region."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ms, units = bench.reduce_timing(10.0 + 5.0 * rank, 16 * 20, world)
        imgs = bench.rank_images("C1", rank)
        gathered = [torch.zeros(imgs.size) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(imgs.ravel().astype(np.float32)))
        out[rank] = (ms, units, [g.numpy() for g in gathered])
    finally:
        dist.destroy_process_group()


def test_reduce_timing_and_distinct_rank_batches():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        ms, units, g = out[r]
        assert ms == pytest.approx(15.0) and units == pytest.approx(2 * 16 * 20)
        assert not np.array_equal(g[0], g[1])          # ranks process different images
        assert np.array_equal(out[0][2][r], out[1][2][r])
