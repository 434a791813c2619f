"""The row split's cross-process peer-memory path on a real GPU.

A row-split call maps every rank's cWY workspace replica into each process with CUDA IPC and
the persistent kernel addresses peer replicas as `own base + delta[k]`.  Two processes (ranks
0 and 1, world_size 2, handles exchanged over torch.distributed `gloo` through the library's
host-exchange hook instead of NCCL, which refuses two ranks on one device) share GPU 0 here:
tinv_debug_peer_map grows the workspace exactly as a row-split call does, exchanges the IPC
handles, opens the peers' mappings and has a kernel read every rank's tag through them.  No
kernel waits on another rank (the cross-rank barrier of the persistent kernel is exercised by
the virtual-rank tests in test_gpu_parity.py, in one cooperative launch).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allgather(send: bytes, nbytes: int) -> bytes:
    outs = [None] * dist.get_world_size()
    dist.all_gather_object(outs, send)
    assert all(len(o) == nbytes for o in outs)
    return b"".join(outs)


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1209_1910_b200.tinv import Tinv, TinvError

        torch.cuda.set_device(0)
        h = Tinv(0, nranks=world, rank=rank, nccl_id=None)
        h.set_host_exchange(_allgather)
        res = []
        # first mapping, then a larger workspace (peers unmap collectively before the free and
        # map the new allocation), then the same size again (mappings reused, new tags)
        for nbytes, base in ((64 << 20, 0xA0), (192 << 20, 0xB0), (128 << 20, 0xC0)):
            res.append(h.debug_peer_map(nbytes, base + rank))
        # without an NCCL communicator the solver refuses multi-rank calls
        try:
            dd = torch.ones(4, dtype=torch.float64, device="cuda:0")
            h.eigvecs(dd, (dd[:3] * 0).contiguous(), dd)
            refused = False
        except TinvError:
            refused = True
        h.close()   # collective: unmaps before the workspace is freed
        np.save(os.path.join(out_dir, f"tags{rank}.npy"), np.array(res, dtype=np.uint64))
        np.save(os.path.join(out_dir, f"refused{rank}.npy"), np.array([refused]))
    finally:
        dist.destroy_process_group()


def test_two_process_ipc_peer_map(tmp_path):
    assert torch.cuda.is_available()
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        tags = np.load(tmp_path / f"tags{r}.npy")
        assert tags.tolist() == [[0xA0, 0xA1], [0xB0, 0xB1], [0xC0, 0xC1]], (r, tags)
        assert bool(np.load(tmp_path / f"refused{r}.npy")[0])
