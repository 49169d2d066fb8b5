"""Host logic of the N > 1 bench path ("replicas only"): two
gloo ranks on CPU run bench.reduce_over_ranks; the job time is the max over
ranks and the work the sum over ranks.  Also checks the bench JSON contract
helpers that need no GPU."""
import os
import socket
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms, applies = bench.reduce_over_ranks(10.0 + 5.0 * rank, 52 + rank, dist, torch.device("cpu"))
    out[rank] = (ms, applies)
    dist.barrier()
    dist.destroy_process_group()


def test_replica_reduction_gloo_ws2():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[0] == out[1] == (15.0, 105)


def test_reduce_single_rank():
    import bench
    assert bench.reduce_over_ranks(3.5, 7) == (3.5, 7)


def test_dist_env_defaults(monkeypatch):
    import bench
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        monkeypatch.delenv(k, raising=False)
    assert bench.dist_env() == (1, 0, 0)


def _groups_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import argparse
    import bench
    args = argparse.Namespace(mode="directions")
    dp = bench.direction_groups(args, world, rank, 4, dist)
    out[rank] = (dp["size"], dp["rank"])
    dist.barrier()
    dist.destroy_process_group()


def test_direction_groups_gloo_ws2():
    """bench --mode directions at N = 2, t = 4: one group of 2 ranks, each owning
    two directions (its local rank 0 / 1)."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_groups_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[0] == (2, 0) and out[1] == (2, 1)


def test_setup_flop_model():
    """The setup roofline's flop model: C5, 33 segments."""
    import bench
    from helm_inputs import make_config
    fl = bench.setup_flops(make_config(5), 33)
    # 2 axes x (2 edge strips of 34 nodes + 30 interior of 35) x 8 w^3 (3 n_c + 4 K + K (K-1))
    per = lambda w: 8.0 * w ** 3 * (3 * 1025 + 4 * 32 + 32 * 31)
    assert abs(fl - 2 * (2 * per(34) + 30 * per(35))) < 1.0
