"""N > 1 path on CPU: two gloo ranks exercise bench.py's max-over-ranks job timing (the only
collective of the replica / weak-scaling bench -- no data-path collective)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    s, fps = bench.job_throughput(1.0 + rank, 3, world, "cpu")
    out[rank] = (s, fps)
    dist.barrier()
    dist.destroy_process_group()


def test_job_throughput_is_max_over_ranks_gloo():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        s, fps = out[r]
        assert s == pytest.approx(2.0)          # slowest rank defines the job time
        assert fps == pytest.approx(2 * 3 / 2.0)  # all ranks' frames / job time


def test_single_rank_throughput():
    import bench
    s, fps = bench.job_throughput(0.5, 2, 1, "cpu")
    assert s == 0.5 and fps == pytest.approx(4.0)
