"""Seeded synthetic workloads (the ONLY module shared by the oracle side and the CUDA side).

It holds no arithmetic of the method (no Riccati, no scan, no linearisation, no line search):
only random problem data with the shapes, structure and value distributions of the paper's
workloads, following the recipes of SURVEY.md §8(d) and DESIGN.md "Input recipe".
Every generator is deterministic in its seed; instance b of a batch draws from
``numpy.random.SeedSequence(seed).spawn(first + B)[first + b]`` so that any slice of a batch
(e.g. one rank's shard) regenerates bit-identically.

All arrays are float64, row-major, batch-outermost, with the conventions of include/pdilqr.h:
  A[B][N+1][n][n] Bm[B][N+1][n][m] c[B][N+1][n] Q[B][N+1][n][n] R[B][N+1][m][m]
  S[B][N+1][m][n] q[B][N+1][n] r[B][N+1][m] P_term[B][n][n] p_term[B][n] dx0[B][n]
SRBD iterate: x[B][N+2][12] u[B][N+1][12] lam[B][N+2][12] x0[B][12] x_ref[B][N+2][12]
  u_ref[B][N+1][12] contact[B][N+1][4] (uint8) feet[B][N+1][4][3].
"""
from __future__ import annotations

import math

import numpy as np

BASE_SEED = 20250609

LQ_KEYS = ("A", "Bm", "c", "Q", "R", "S", "q", "r", "P_term", "p_term", "dx0")


def _rngs(seed: int, B: int, first: int = 0):
    ss = np.random.SeedSequence(seed).spawn(first + B)[first:]
    return [np.random.default_rng(s) for s in ss]


# --------------------------------------------------------------------------------------
# Config 1: time-invariant double integrator, n=4 m=2
# --------------------------------------------------------------------------------------
def double_integrator(N: int = 32, dt: float = 0.1, variant: str = "kkt", seed: int = BASE_SEED):
    """Config 1.  A=[[I,dt I],[0,I]], B=[[0],[dt I]], Q=I4, R=0.1 I2, S=0.

    variant "dare": q=r=b=0 and P_term=Q (the DARE test overrides P_term with P_inf);
    variant "kkt":  q, r, b ~ N(0, 0.1^2), P_term = Q.   dx0 = (1, -1, 0.5, 0).
    Batch size 1.
    """
    n, m = 4, 2
    I2 = np.eye(2)
    A = np.block([[I2, dt * I2], [np.zeros((2, 2)), I2]])
    Bm = np.vstack([np.zeros((2, 2)), dt * I2])
    rng = _rngs(seed, 1)[0]
    S1 = N + 1
    qp = {
        "A": np.broadcast_to(A, (1, S1, n, n)).copy(),
        "Bm": np.broadcast_to(Bm, (1, S1, n, m)).copy(),
        "Q": np.broadcast_to(np.eye(n), (1, S1, n, n)).copy(),
        "R": np.broadcast_to(0.1 * np.eye(m), (1, S1, m, m)).copy(),
        "S": np.zeros((1, S1, m, n)),
        "P_term": np.eye(n)[None].copy(),
        "p_term": np.zeros((1, n)),
        "dx0": np.array([[1.0, -1.0, 0.5, 0.0]]),
    }
    if variant == "dare":
        qp["c"] = np.zeros((1, S1, n))
        qp["q"] = np.zeros((1, S1, n))
        qp["r"] = np.zeros((1, S1, m))
    else:
        qp["c"] = 0.1 * rng.standard_normal((1, S1, n))
        qp["q"] = 0.1 * rng.standard_normal((1, S1, n))
        qp["r"] = 0.1 * rng.standard_normal((1, S1, m))
        qp["p_term"] = 0.1 * rng.standard_normal((1, n))
    return qp


# --------------------------------------------------------------------------------------
# Random LQ problems
# --------------------------------------------------------------------------------------
def _spectral_rescale(M):
    rho = np.max(np.abs(np.linalg.eigvals(M)))
    return M / rho if rho > 0 else M


def random_lq(B: int, N: int, n: int, m: int, seed: int = BASE_SEED, first: int = 0,
              kind: str = "dense", dt: float = 0.01):
    """Random well-posed LQ subproblems of Eq. 4 (Q PSD, R SPD, [[Q,S^T],[S,R]] PSD).

    kind "dense": A = I + 0.1 G/sqrt(n) (G standard normal), B ~ N(0, 1/m), Q = dense SPD with
        eigenvalues U[0.1, 10], R = dense SPD with eigenvalues U[0.1, 2], S small, q, r, c ~
        N(0, 0.1^2), P_term = dense SPD, dx0 ~ N(0, 1).  Exercises every block of the element
        algebra (full C, P, A; nonzero S).
    kind "wb": config-5 recipe: second-order structure
        A = [[I, dt I], [dt Fq, I + dt Fv]], B = [[0], [dt G]], Q = diag U[0.1, 10],
        R = diag U[1e-3, 1e-1], ||S||_2 <= 0.1 sqrt(lmin(Q) lmin(R)), q, r, c ~ N(0, 0.1^2),
        P_term = 10 Q_N, each stage perturbed by 1% (time-varying).  Needs even n.
    """
    S1 = N + 1
    out = {k: None for k in LQ_KEYS}
    A = np.empty((B, S1, n, n)); Bm = np.empty((B, S1, n, m)); c = np.empty((B, S1, n))
    Q = np.empty((B, S1, n, n)); R = np.empty((B, S1, m, m)); S = np.empty((B, S1, m, n))
    q = np.empty((B, S1, n)); r = np.empty((B, S1, m)); Pt = np.empty((B, n, n))
    pt = np.empty((B, n)); dx0 = np.empty((B, n))
    for b, rng in enumerate(_rngs(seed, B, first)):
        if kind == "wb":
            assert n % 2 == 0
            nq = n // 2
            Fq = _spectral_rescale(rng.standard_normal((nq, nq)) / math.sqrt(nq))
            Fv = _spectral_rescale(rng.standard_normal((nq, nq)) / math.sqrt(nq))
            G = rng.standard_normal((nq, m)) / math.sqrt(m)
            A0 = np.block([[np.eye(nq), dt * np.eye(nq)], [dt * Fq, np.eye(nq) + dt * Fv]])
            B0 = np.vstack([np.zeros((nq, m)), dt * G])
            qd = rng.uniform(0.1, 10.0, n)
            rd = rng.uniform(1e-3, 1e-1, m)
            for i in range(S1):
                A[b, i] = A0 * (1.0 + 0.01 * rng.standard_normal((n, n)))
                Bm[b, i] = B0 * (1.0 + 0.01 * rng.standard_normal((n, m)))
                Qi = np.diag(qd * (1.0 + 0.01 * rng.uniform(-1, 1, n)))
                Ri = np.diag(rd * (1.0 + 0.01 * rng.uniform(-1, 1, m)))
                Si = rng.standard_normal((m, n))
                Si *= 0.1 * math.sqrt(Qi.diagonal().min() * Ri.diagonal().min()) / np.linalg.norm(Si, 2)
                Q[b, i], R[b, i], S[b, i] = Qi, Ri, Si
            Pt[b] = 10.0 * Q[b, N]
        else:
            for i in range(S1):
                A[b, i] = np.eye(n) + 0.1 * rng.standard_normal((n, n)) / math.sqrt(n)
                Bm[b, i] = rng.standard_normal((n, m)) / math.sqrt(m)
                U, _ = np.linalg.qr(rng.standard_normal((n, n)))
                Qi = (U * rng.uniform(0.1, 10.0, n)) @ U.T
                V, _ = np.linalg.qr(rng.standard_normal((m, m)))
                Ri = (V * rng.uniform(0.1, 2.0, m)) @ V.T
                Si = rng.standard_normal((m, n))
                Si *= 0.2 * math.sqrt(0.1 * 0.1) / max(np.linalg.norm(Si, 2), 1e-300)
                Q[b, i], R[b, i], S[b, i] = 0.5 * (Qi + Qi.T), 0.5 * (Ri + Ri.T), Si
            W, _ = np.linalg.qr(rng.standard_normal((n, n)))
            Ptb = (W * rng.uniform(0.1, 10.0, n)) @ W.T
            Pt[b] = 0.5 * (Ptb + Ptb.T)
        c[b] = 0.1 * rng.standard_normal((S1, n))
        q[b] = 0.1 * rng.standard_normal((S1, n))
        r[b] = 0.1 * rng.standard_normal((S1, m))
        pt[b] = 0.1 * rng.standard_normal(n)
        dx0[b] = rng.standard_normal(n)
    out.update(A=A, Bm=Bm, c=c, Q=Q, R=R, S=S, q=q, r=r, P_term=Pt, p_term=pt, dx0=dx0)
    return out


# --------------------------------------------------------------------------------------
# SRBD quadruped MPC workload (configs 2 and 3)
# --------------------------------------------------------------------------------------
def srbd_default_params() -> dict:
    """SRBD model / cost parameters (reading R15: only the 15 kg mass is from the paper, P:375;
    the rest are recorded choices).  Field names follow pdilqr_srbd_params."""
    return {
        "dt": 0.02,                                   # 50 Hz (reading R14)
        "mass": 15.0,                                 # Go2
        "inertia": [0.10, 0.0, 0.0, 0.0, 0.25, 0.0, 0.0, 0.0, 0.28],
        "gravity": [0.0, 0.0, -9.81],
        # state weights: p(3), Theta(3), v(3), w(3)
        "w_x": [10.0, 10.0, 500.0, 100.0, 100.0, 50.0, 5.0, 5.0, 10.0, 1.0, 1.0, 1.0],
        "w_x_term": [50.0, 50.0, 2500.0, 500.0, 500.0, 250.0, 25.0, 25.0, 50.0, 5.0, 5.0, 5.0],
        "w_u_stance": 1e-3,
        "w_u_swing": 10.0,
        "mu_friction": 0.6,
        "f_min": 2.0,
        "f_max": 250.0,
        "barrier_mu": 0.1,
        "barrier_delta": 1.0,
    }


HIP_OFFSETS = np.array([[0.19, 0.12], [0.19, -0.12], [-0.19, 0.12], [-0.19, -0.12]])  # FL FR RL RR
NOMINAL_HEIGHT = 0.30
GAIT_PERIOD = 0.4        # s: trot, 10 stages per half period at dt = 0.02


def _rotz(yaw):
    c, s = math.cos(yaw), math.sin(yaw)
    return np.array([[c, -s], [s, c]])


def _ref_pos(p0, yaw0, wz, vb, t):
    """Reference CoM xy at times t (array) for a constant body-frame velocity vb and yaw rate wz:
    p0 + int_0^t Rz(yaw0 + wz s) vb ds (closed form).  Returns [len(t)][2]."""
    t = np.asarray(t, dtype=np.float64)
    if abs(wz) < 1e-9:
        return p0[None, :] + t[:, None] * (_rotz(yaw0) @ vb)[None, :]
    s0, c0 = math.sin(yaw0), math.cos(yaw0)
    s1, c1 = np.sin(yaw0 + wz * t), np.cos(yaw0 + wz * t)
    ic, is_ = (s1 - s0) / wz, (c0 - c1) / wz            # int cos, int sin
    return p0[None, :] + np.stack([ic * vb[0] - is_ * vb[1], is_ * vb[0] + ic * vb[1]], axis=1)


def srbd_problem(B: int, N: int = 50, seed: int = BASE_SEED, first: int = 0, params: dict | None = None,
                 randomize: bool = True, v_cmd=(0.5, 0.0)):
    """SRBD trot MPC instances (configs 2/3).

    Config 2 (``randomize=False``): v_cmd = (0.5, 0) m/s (overridable), yaw rate 0, gait phase 0.
    Config 3 (``randomize=True``): per instance v_cmd ~ U(-0.5, 0.5)^2, yaw rate ~ U(-0.5, 0.5),
    gait phase ~ U(0, 1), initial yaw ~ U(-pi, pi), initial xy ~ U(-1, 1)^2.
    Diagonal trot (FL+RR / FR+RL), period 0.4 s, duty 0.5; footholds at mid-stance hip positions
    of the reference (Raibert-style, SPEC S:397/S:467 -- host-side input generation only).
    x_hat0 = x_ref[0] + N(0, sigma) with sigma_p=0.02, sigma_Theta=0.05, sigma_v=0.1, sigma_w=0.1.
    Iterate: x = x_ref, u = u_ref (gravity split over stance feet), lam = 0 (cold start).
    """
    prm = srbd_default_params() if params is None else params
    dt, mass, g = prm["dt"], prm["mass"], -prm["gravity"][2]
    S1, S2 = N + 1, N + 2
    x_ref = np.zeros((B, S2, 12)); u_ref = np.zeros((B, S1, 12))
    contact = np.zeros((B, S1, 4), dtype=np.uint8); feet = np.zeros((B, S1, 4, 3))
    x0 = np.zeros((B, 12))
    t_nodes = dt * np.arange(S2)
    for b, rng in enumerate(_rngs(seed, B, first)):
        if randomize:
            vcmd = rng.uniform(-0.5, 0.5, 2); wz = rng.uniform(-0.5, 0.5)
            phase = rng.uniform(0.0, 1.0); yaw0 = rng.uniform(-math.pi, math.pi)
            p0 = rng.uniform(-1.0, 1.0, 2)
        else:
            vcmd = np.array(v_cmd, dtype=np.float64); wz = 0.0; phase = 0.0; yaw0 = 0.0; p0 = np.zeros(2)
        yaw = yaw0 + wz * t_nodes
        cy, sy = np.cos(yaw), np.sin(yaw)
        vel = np.stack([cy * vcmd[0] - sy * vcmd[1], sy * vcmd[0] + cy * vcmd[1]], axis=1)  # world xy
        pos = p0 + np.concatenate([np.zeros((1, 2)), np.cumsum(vel[:-1] * dt, axis=0)])
        x_ref[b, :, 0:2] = pos
        x_ref[b, :, 2] = NOMINAL_HEIGHT
        x_ref[b, :, 5] = yaw
        x_ref[b, :, 6:8] = vel
        x_ref[b, :, 11] = wz
        # gait: pair A = {FL, RR} stands while s < 0.5, pair B = {FR, RL} otherwise
        s = (phase + t_nodes[:S1] / GAIT_PERIOD) % 1.0
        pairA = s < 0.5
        contact[b, :, 0] = pairA; contact[b, :, 3] = pairA
        contact[b, :, 1] = ~pairA; contact[b, :, 2] = ~pairA
        # footholds: hip position of the reference at the middle of the stance phase that
        # contains (or, for swing stages, follows) stage i
        cyc = phase + t_nodes[:S1] / GAIT_PERIOD
        for j in range(4):
            in_a = j in (0, 3)
            start = np.floor(cyc) + (0.0 if in_a else 0.5)
            start = np.where(start > cyc, start - 1.0, start)
            start = np.where(cyc - start >= 0.5, start + 1.0, start)   # in swing: next stance phase
            t_mid = (start + 0.25 - phase) * GAIT_PERIOD
            yaw_m = yaw0 + wz * t_mid
            p_m = _ref_pos(p0, yaw0, wz, vcmd, t_mid)                # reference CoM at mid-stance
            hx, hy = HIP_OFFSETS[j]
            feet[b, :, j, 0] = p_m[:, 0] + np.cos(yaw_m) * hx - np.sin(yaw_m) * hy
            feet[b, :, j, 1] = p_m[:, 1] + np.sin(yaw_m) * hx + np.cos(yaw_m) * hy
            feet[b, :, j, 2] = 0.0
        nst = np.maximum(contact[b].sum(axis=1), 1).astype(np.float64)
        u_ref[b, :, 2::3] = contact[b] * (mass * g / nst)[:, None]
        sig = np.array([0.02] * 3 + [0.05] * 3 + [0.1] * 3 + [0.1] * 3)
        x0[b] = x_ref[b, 0] + sig * rng.standard_normal(12)
    x = x_ref.copy()
    u = u_ref.copy()
    lam = np.zeros((B, S2, 12))
    return {
        "params": prm, "N": N,
        "x": x, "u": u, "lam": lam, "x0": x0, "x_ref": x_ref, "u_ref": u_ref,
        "contact": contact, "feet": feet,
    }


def round_to(arrs: dict, dtype) -> dict:
    """Round every floating array to ``dtype`` and back to float64 (the rounded
    values are what both sides consume, so input quantisation is not counted as GPU error)."""
    out = {}
    for k, v in arrs.items():
        if isinstance(v, np.ndarray) and v.dtype == np.float64:
            out[k] = v.astype(dtype).astype(np.float64)
        else:
            out[k] = v
    return out


# --------------------------------------------------------------------------------------
# Config 4: centralized controller for R quadrupeds (NEXT-3 model)
# --------------------------------------------------------------------------------------
def multi_default_params(n_robots: int = 16) -> dict:
    """Collision-penalty parameters of the centralized model (recorded choices: the paper gives
    only "a quadratic penalty term"): d_min = 1.0 m, weight 1e3, softplus sharpness 10 /m."""
    return {"n_robots": n_robots, "d_min": 1.0, "weight": 1.0e3, "sharpness": 10.0}


def multi_srbd_problem(B: int, n_robots: int = 16, N: int = 50, seed: int = BASE_SEED, first: int = 0,
                       spacing: float = 1.5, multi: dict | None = None):
    """Config 4: R SRBD robots (config-3 trot instances: random commands, phases and yaw) on a
    ceil(sqrt R) x ceil(sqrt R) grid `spacing` metres apart (4 x 4, 1.5 m for R = 16), stacked
    robot by robot into one instance: x[B][N+2][12R], u[B][N+1][12R], lam, x0[B][12R],
    x_ref, u_ref, contact[B][N+1][4R], feet[B][N+1][4R][3].  Robot k of instance b is the
    config-3 draw number first * R + b * R + k; only the grid offsets of positions, references and
    footholds are added here (data generation, no method arithmetic)."""
    R = n_robots
    one = srbd_problem(B * R, N=N, seed=seed, first=first * R)
    side = int(math.ceil(math.sqrt(R)))
    S1, S2 = N + 1, N + 2
    out = {"params": one["params"], "multi": multi or multi_default_params(R), "N": N}
    for key, shp in (("x", (S2, 12)), ("u", (S1, 12)), ("lam", (S2, 12)), ("x_ref", (S2, 12)), ("u_ref", (S1, 12))):
        a = one[key].reshape(B, R, *shp).copy()
        if key in ("x", "x_ref"):
            for k in range(R):
                a[:, k, :, 0] += spacing * (k % side)
                a[:, k, :, 1] += spacing * (k // side)
        out[key] = np.ascontiguousarray(np.moveaxis(a, 1, 2).reshape(B, shp[0], 12 * R))
    x0 = one["x0"].reshape(B, R, 12).copy()
    feet = one["feet"].reshape(B, R, S1, 4, 3).copy()
    for k in range(R):
        x0[:, k, 0] += spacing * (k % side)
        x0[:, k, 1] += spacing * (k // side)
        feet[:, k, :, :, 0] += spacing * (k % side)
        feet[:, k, :, :, 1] += spacing * (k // side)
    out["x0"] = np.ascontiguousarray(x0.reshape(B, 12 * R))
    out["feet"] = np.ascontiguousarray(np.moveaxis(feet, 1, 2).reshape(B, S1, 4 * R, 3))
    out["contact"] = np.ascontiguousarray(np.moveaxis(one["contact"].reshape(B, R, S1, 4), 1, 2).reshape(B, S1, 4 * R))
    return out

