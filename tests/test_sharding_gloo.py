"""Multi-process logic of the batch-sharded bench on CPU with gloo, world_size 2,
through the same functions bench.py calls (paper_2506_07823_b200/sharding.py): each rank
regenerates only its own instances [r*B, (r+1)*B) and solves them (the fp64 oracle stands in for
the GPU solver), then one all_gather assembles u0 and the stats; the result must equal the
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
    from paper_2506_07823_b200 import sharding
    first, nb = sharding.shard(BPR, rank)
    prob = synth.srbd_problem(nb, N=N, seed=synth.BASE_SEED, first=first)
    st = O.srbd_step(prob, nthreads=1)          # the fp64 oracle stands in for the GPU step
    stats = {k: torch.from_numpy(st[:, j].copy()) for j, k in enumerate(sharding.STAT_KEYS)}
    packed = sharding.pack_results(torch.from_numpy(prob["u"][:, 0, :].copy()), stats)
    g = sharding.gather_results(packed, WORLD, dist)
    tmax = sharding.max_over_ranks(float(rank + 1), WORLD, torch.device("cpu"), dist)
    if rank == 0:
        np.savez(out_path, g=g.numpy(), tmax=np.array([tmax]))
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
    assert np.array_equal(g["g"][:, :12], full["u"][:, 0, :])
    assert np.array_equal(g["g"][:, 12:], st)
    assert g["tmax"][0] == WORLD


def test_rank_slices_regenerate_bitwise():
    full = synth.srbd_problem(6, N=5, seed=7)
    part = synth.srbd_problem(2, N=5, seed=7, first=3)
    for k in ("x", "u", "x0", "x_ref", "feet", "contact"):
        assert np.array_equal(full[k][3:5], part[k])


def test_horizon_split_covers_stages():
    from paper_2506_07823_b200 import horizon
    for N in (0, 1, 7, 50, 1000):
        for G in (1, 2, 3, 8):
            ch = horizon.split_stages(N, G)
            assert ch[0][0] == 0 and ch[-1][1] == N + 1
            assert all(a[1] == b[0] for a, b in zip(ch, ch[1:]))
            sizes = [e - s for s, e in ch]
            assert max(sizes) - min(sizes) <= 1


def _gather_worker(rank, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_2506_07823_b200 import horizon
    g = horizon.dist_all_gather(dist)(torch.full((3, 5), float(rank)))
    if rank == 0:
        np.save(out_path, g.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_horizon_all_gather_gloo(tmp_path):
    """The collective of the horizon-sharded solve (horizon.dist_all_gather): rank-major stacking."""
    out = str(tmp_path / "g.npy")
    mp.spawn(_gather_worker, args=(_free_port(), out), nprocs=WORLD, join=True)
    g = np.load(out)
    assert g.shape == (WORLD, 3, 5) and (g[0] == 0).all() and (g[1] == 1).all()
