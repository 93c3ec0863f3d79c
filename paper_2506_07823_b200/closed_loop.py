"""Closed-loop RTI on the GPU (Table I).

Each control tick, for all B environments at once:
  1. x0 <- plant state                                (torch copy, plumbing)
  2. one SQP iteration           pdilqr_step           ("one iteration only of the algorithm")
  then for each of the k nodes until the next tick (plan playback):
  3. plant: RK4 of the SRBD model over dt              pdilqr_srbd_plant, u_0 held
  4. warm start: shift by one node                     pdilqr_shift ("shifted by one time-step")
  5. slide the reference window by one node           (torch copy, plumbing)
k = nodes per tick (1 -> control at 1/dt = 50 Hz, 2 -> 25 Hz with the same 20 ms MPC nodes).
All compute is in libpdilqr.so; this module only sequences calls and copies windows.
"""
from __future__ import annotations

import contextlib

import torch

from .pdilqr import PDILQR_MODEL_SRBD, PdIlqr


class ClosedLoop:
    """B environments, each with its own MPC (Table I).  `ref` holds device tensors for a long
    horizon: x_ref [B, L+2, 12], u_ref [B, L+1, 12], contact [B, L+1, 4] u8, feet [B, L+1, 4, 3],
    L >= N + k * ticks.  `it0` is the initial iterate (x, u, lam windows of length N+2/N+1/N+2)."""

    def __init__(self, h: PdIlqr, ref: dict, it0: dict, x_plant0: torch.Tensor, nodes_per_tick: int = 1,
                 substeps: int = 4):
        if h._cfg.model != PDILQR_MODEL_SRBD:
            raise ValueError("closed loop needs an SRBD handle")
        self.h, self.ref, self.k, self.sub = h, ref, int(nodes_per_tick), int(substeps)
        self.N = h.N
        self.dt = float(h._cfg.srbd.dt)
        self.t = 0
        self.node = 0
        N = self.N
        self.it = {k: it0[k].clone().contiguous() for k in ("x", "u", "lam")}
        self.it["x0"] = x_plant0.clone().contiguous()
        for k, L in (("x_ref", N + 2), ("u_ref", N + 1), ("contact", N + 1), ("feet", N + 1)):
            self.it[k] = ref[k][:, :L].clone().contiguous()
        self.x_plant = x_plant0.clone().contiguous()
        self.u_hold = torch.empty_like(self.x_plant)
        self.stats = h.new_stats()

    @property
    def horizon_left(self) -> int:
        return (self.ref["x_ref"].shape[1] - 2) - (self.N + self.node)

    def _window(self):
        N, o = self.N, self.node
        self.it["x_ref"].copy_(self.ref["x_ref"][:, o:o + N + 2])
        for key in ("u_ref", "contact", "feet"):
            self.it[key].copy_(self.ref[key][:, o:o + N + 1])

    def tick(self, ext_force=None, stream=None) -> dict:
        """One control tick: x0 <- plant, one SQP iteration, then k nodes of plant + shift + window
        slide (plan playback between ticks).  ext_force: None, a [B,3] tensor, or a callable
        node -> tensor/None.  Returns the stats dict of the SQP iteration (device tensors)."""
        if self.horizon_left < self.k:
            raise RuntimeError("reference horizon exhausted")
        # every copy and every library call of the tick on one stream (the caller's, else torch's
        # current one), so the x0 / u_hold / window copies are ordered with step, plant and shift
        ctx = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
        with ctx:
            s = torch.cuda.current_stream(self.x_plant.device)
            self.it["x0"].copy_(self.x_plant)
            self.h.step(self.it, self.stats, stream=s)
            for _ in range(self.k):
                F = ext_force(self.node) if callable(ext_force) else ext_force
                self.u_hold.copy_(self.it["u"][:, 0])
                self.h.plant(self.it, self.x_plant, self.u_hold, F, dt=self.dt, substeps=self.sub, stream=s)
                self.h.shift(self.it, stream=s)
                self.node += 1
                self._window()
        self.t += 1
        return self.stats
