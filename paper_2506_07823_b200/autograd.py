"""Differentiable LQ solve (NEXT-4 of SURVEY §8(f); the "learning" use of the solver, P:61-62,
P:317): a torch.autograd.Function whose forward is pdilqr_solve_lq and whose backward is
pdilqr_solve_lq_adjoint (one more pass of the same parallel scans + outer products, all in the
library's kernels).  Argument marshalling only.

    dx, du, dlam = lq_solve(handle, qp)          # qp: dict of the 11 Eq. 4 tensors
    loss(dx, du, dlam).backward()                # gradients land in qp[k].grad
"""
from __future__ import annotations

import torch

KEYS = ("A", "Bm", "c", "Q", "R", "S", "q", "r", "P_term", "p_term", "dx0")


class LqSolveFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, handle, *tensors):
        qp = dict(zip(KEYS, tensors))
        out = handle.solve_lq(qp)
        ctx.handle = handle
        ctx.save_for_backward(*tensors, out["dx"], out["du"], out["dlam"])
        ctx.mark_non_differentiable(out["info"])
        return out["dx"], out["du"], out["dlam"], out["info"]

    @staticmethod
    def backward(ctx, gdx, gdu, gdlam, _ginfo):
        saved = ctx.saved_tensors
        qp = dict(zip(KEYS, saved[:len(KEYS)]))
        sol = {"dx": saved[-3], "du": saved[-2], "dlam": saved[-1]}
        gs = {k: (None if g is None else g.contiguous()) for k, g in (("dx", gdx), ("du", gdu), ("dlam", gdlam))}
        want = [k for k, need in zip(KEYS, ctx.needs_input_grad[1:]) if need]
        h = ctx.handle
        shapes = h.lq_shapes()
        grad = {k: torch.empty(shapes[k], dtype=h.dtype, device=h.device) for k in want}
        grad = h.solve_lq_adjoint(qp, sol, gs, grad)
        return (None,) + tuple(grad.get(k) for k in KEYS)


def lq_solve(handle, qp: dict):
    """Differentiable pdilqr_solve_lq: returns (dx, du, dlam, info)."""
    return LqSolveFunction.apply(handle, *[qp[k].contiguous() for k in KEYS])
