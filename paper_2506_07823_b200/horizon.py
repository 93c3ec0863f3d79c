"""Horizon-sharded LQ solve over ranks (NEXT-2 of SURVEY §8(f)): one long-horizon problem split into
G contiguous stage chunks, one per rank (one process per GPU), exact by the associativity of the
scan elements (Eq. 8).  Per rank: chunk reduce -> all-gather of the chunk summaries ->
local suffix -> local backward solve -> all-gather of the chunk's closed-loop map -> local prefix ->
local rollout.  Two all-gathers of O(n^2) values per instance; every arithmetic step runs in the
library's kernels (include/pdilqr.h, pdilqr_lq_segment_*).  Plumbing only.

    out = solve_lq_sharded(handle, qp_local, P_term, p_term, dx0, rank, world, all_gather)

`qp_local` holds this rank's stages (its P_term / p_term / dx0 entries are ignored); `P_term`,
`p_term`, `dx0` are the global problem's.  `all_gather(t) -> tensor [world, *t.shape]` is the
collective (NCCL all_gather_into_tensor on GPUs; gloo through host copies in tests).
"""
from __future__ import annotations

import torch


def split_stages(N_global: int, world: int) -> list[tuple[int, int]]:
    """Contiguous chunks [s_r, e_r) of the N_global + 1 stages, sizes differing by at most one."""
    L = N_global + 1
    base, extra = divmod(L, world)
    out, s = [], 0
    for r in range(world):
        e = s + base + (1 if r < extra else 0)
        out.append((s, e))
        s = e
    return out


def local_problem(qp: dict, s: int, e: int) -> dict:
    """Stages [s, e) of a global Eq. 4 dict (batch-outermost) as a local LQ dict (P_term, p_term, dx0
    placeholders zero)."""
    loc = {k: qp[k][:, s:e].contiguous() for k in ("A", "Bm", "c", "Q", "R", "S", "q", "r")}
    B, n = qp["dx0"].shape
    loc["P_term"] = torch.zeros_like(qp["P_term"])
    loc["p_term"] = torch.zeros_like(qp["p_term"])
    loc["dx0"] = torch.zeros_like(qp["dx0"])
    return loc


def dist_all_gather(dist, device=None):
    """all_gather for torch.distributed: NCCL on CUDA tensors, else through host tensors (gloo)."""
    def gather(t):
        world = dist.get_world_size()
        src = t if device is None else t.to(device)
        out = torch.empty((world * src.shape[0],) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
        dist.all_gather_into_tensor(out, src.contiguous())
        return out.view((world,) + tuple(src.shape)).to(t.device)
    return gather


def solve_lq_sharded(h, qp_local: dict, P_term, p_term, dx0, rank: int, world: int, all_gather) -> dict:
    S = h.segment_reduce(qp_local)
    S_all = all_gather(S)
    Pe, pe = h.segment_suffix(S_all, rank, P_term, p_term)
    qp = dict(qp_local, P_term=Pe, p_term=pe, dx0=torch.zeros_like(dx0))
    out = h.solve_lq(qp)
    F = h.segment_forward(qp)
    F_all = all_gather(F)
    qp["dx0"] = h.segment_prefix(F_all, rank, dx0)
    return h.solve_lq(qp, out=out)
