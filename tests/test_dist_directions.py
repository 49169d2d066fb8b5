"""Host logic of the direction-parallel solve (mpgmres_solve_dist)
on CPU: the direction split, and the all-gather callback the binding hands to
the C ABI, run by two gloo ranks on host buffers (in place, rank order)."""
import ctypes
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2408_11929_b200 as hs


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partition_directions():
    assert hs.partition_directions(["LRL", "RLR", "BTB", "TBT"], 2) == [["LRL", "RLR"], ["BTB", "TBT"]]
    assert hs.partition_directions(["LRL", "RLR", "BTB", "TBT"], 4) == [["LRL"], ["RLR"], ["BTB"], ["TBT"]]
    assert hs.partition_directions(["LRL", "BTB"], 1) == [["LRL", "BTB"]]
    with pytest.raises(ValueError):
        hs.partition_directions(["LRL", "RLR", "BTB"], 2)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, tl = 7, 2                                   # 2 local columns of 7 complex values
    recv = np.zeros(world * tl * n, dtype=np.complex128)
    mine = recv[rank * tl * n:(rank + 1) * tl * n]
    mine[:] = (rank + 1) * (np.arange(tl * n) + 1j)
    cb = hs.torch_allgather(device=False)
    nbytes = tl * n * 16
    rc = cb(None, mine.ctypes.data, recv.ctypes.data, nbytes, None)
    out[rank] = (rc, recv.copy())
    dist.barrier()
    dist.destroy_process_group()


def test_allgather_callback_gloo_ws2():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    n, tl = 7, 2
    expect = np.concatenate([(r + 1) * (np.arange(tl * n) + 1j) for r in range(2)])
    for r in range(2):
        rc, recv = out[r]
        assert rc == 0
        assert np.array_equal(recv, expect)
