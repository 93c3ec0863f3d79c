"""Multi-process logic of the batch-sharded bench on CPU with gloo, world_size 2:
each rank regenerates only its own instances [r*B, (r+1)*B) and solves them (the fp64 oracle stands
in for the GPU solver), then one all_gather assembles u0 and the stats; the result must equal the
single-process run on the full batch."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from workloads import synth

BPR, N, WORLD = 3, 6, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from oracle import oracle as O
    prob = synth.srbd_problem(BPR, N=N, seed=synth.BASE_SEED, first=rank * BPR)
    st = O.srbd_step(prob, nthreads=1)
    u0 = torch.from_numpy(prob["u"][:, 0, :].copy())
    stt = torch.from_numpy(st)
    gu = [torch.empty_like(u0) for _ in range(WORLD)]
    gs = [torch.empty_like(stt) for _ in range(WORLD)]
    dist.all_gather(gu, u0)
    dist.all_gather(gs, stt)
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)      # max-over-ranks timing reduction
    if rank == 0:
        np.savez(out_path, u0=torch.cat(gu).numpy(), st=torch.cat(gs).numpy(), tmax=t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shard_and_gather(tmp_path):
    from oracle import oracle as O
    O.build()
    out = str(tmp_path / "g.npz")
    mp.spawn(_worker, args=(_free_port(), out), nprocs=WORLD, join=True)
    g = np.load(out)
    full = synth.srbd_problem(WORLD * BPR, N=N, seed=synth.BASE_SEED)
    st = O.srbd_step(full, nthreads=1)
    assert np.array_equal(g["u0"], full["u"][:, 0, :])
    assert np.array_equal(g["st"], st)
    assert g["tmax"][0] == WORLD


def test_rank_slices_regenerate_bitwise():
    full = synth.srbd_problem(6, N=5, seed=7)
    part = synth.srbd_problem(2, N=5, seed=7, first=3)
    for k in ("x", "u", "x0", "x_ref", "feet", "contact"):
        assert np.array_equal(full[k][3:5], part[k])
