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
