"""ctypes wrapper of the fp64 CPU oracle (oracle/pdilqr_oracle.c).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports this module, and this
module never imports the product package.  Argument marshalling only; all arithmetic is in C.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pdilqr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


_FLAGS = ["-std=gnu11", "-O3", "-fopenmp", "-fPIC", "-shared", "-Wall"]
_native = False


def build(force: bool = False, native: bool = False) -> str:
    """Compile liboracle.so with gcc (-O3, OpenMP): plain x86-64 code, so the same binary runs on
    any host (tests).  native=True builds liboracle_native.so with -march=native for the timed
    CPU baseline, on the host that runs it (bench.py)."""
    lib = _LIB.replace(".so", "_native.so") if native else _LIB
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *_FLAGS, *(["-march=native"] if native else []), "-o", lib + ".tmp", _SRC])
        os.replace(lib + ".tmp", lib)
    return lib


def use_native() -> None:
    """Timed baselines: load the -march=native build (call before the first oracle call)."""
    global _native
    if _lib is None:
        _native = True


def build_flags() -> str:
    return "gcc " + " ".join(_FLAGS[:3] + (["-march=native"] if _native else []))


class SrbdParams(C.Structure):
    _fields_ = [("dt", C.c_double), ("mass", C.c_double), ("inertia", C.c_double * 9),
                ("gravity", C.c_double * 3), ("w_x", C.c_double * 12), ("w_x_term", C.c_double * 12),
                ("w_u_stance", C.c_double), ("w_u_swing", C.c_double), ("mu_friction", C.c_double),
                ("f_min", C.c_double), ("f_max", C.c_double), ("barrier_mu", C.c_double),
                ("barrier_delta", C.c_double)]

    @classmethod
    def from_dict(cls, d: dict) -> "SrbdParams":
        p = cls()
        for name, _ in cls._fields_:
            v = d[name]
            if isinstance(v, (list, tuple, np.ndarray)):
                arr = getattr(p, name)
                for i, e in enumerate(v):
                    arr[i] = float(e)
            else:
                setattr(p, name, float(v))
        return p


class MultiParams(C.Structure):
    _fields_ = [("n_robots", C.c_int), ("d_min", C.c_double), ("weight", C.c_double), ("sharpness", C.c_double)]

    @classmethod
    def from_dict(cls, d: dict) -> "MultiParams":
        return cls(int(d["n_robots"]), float(d["d_min"]), float(d["weight"]), float(d["sharpness"]))


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build(native=_native))
        i, d, PP = C.c_int, C.c_double, C.POINTER(SrbdParams)
        L.oracle_riccati.argtypes = [i, i, i] + [_dp] * 11 + [_dp] * 4
        L.oracle_riccati.restype = i
        L.oracle_rollout_dual.argtypes = [i, i, i] + [_dp] * 8 + [_dp] * 3
        L.oracle_solve_lq.argtypes = [i, i, i] + [_dp] * 11 + [_dp] * 3 + [_dp] * 4
        L.oracle_solve_lq.restype = i
        L.oracle_solve_lq_batch.argtypes = [i, i, i, i] + [_dp] * 11 + [_dp] * 3 + [_ip, i]
        L.oracle_solve_lq_adjoint.argtypes = [i, i, i] + [_dp] * 6 + [_dp] * 3 + [_dp] * 3 + [_dp] * 11
        L.oracle_solve_lq_adjoint.restype = i
        L.oracle_srbd_f.argtypes = [PP, _dp, _dp, _dp, _up, _dp]
        L.oracle_srbd_jac.argtypes = [PP, _dp, _dp, _dp, _up, _dp, _dp]
        L.oracle_srbd_h.argtypes = [PP, _dp, _dp, _dp, _up, _dp]
        for f in ("oracle_barrier", "oracle_barrier_d1", "oracle_barrier_d2"):
            getattr(L, f).argtypes = [d, d, d]
            getattr(L, f).restype = d
        L.oracle_srbd_linearize.argtypes = [PP, i] + [_dp] * 6 + [_up, _dp] + [_dp] * 11
        L.oracle_srbd_linearize.restype = i
        L.oracle_srbd_linearize_batch.argtypes = [PP, i, i] + [_dp] * 6 + [_up, _dp] + [_dp] * 11 + [_ip, i]
        L.oracle_srbd_cost.argtypes = [PP, i, _dp, _dp, _dp, _dp, _up]
        L.oracle_srbd_cost.restype = d
        L.oracle_srbd_theta.argtypes = [PP, i, _dp, _dp, _dp, _up, _dp]
        L.oracle_srbd_theta.restype = d
        L.oracle_srbd_cost_slope.argtypes = [PP, i, _dp, _dp, _dp, _dp, _up, _dp, _dp]
        L.oracle_srbd_cost_slope.restype = d
        L.oracle_srbd_line_search.argtypes = [PP, i, i, d, d] + [_dp] * 5 + [_up, _dp, _dp, _dp] + [_dp] * 3
        L.oracle_srbd_line_search.restype = i
        L.oracle_srbd_step.argtypes = [PP, i, i, d, d] + [_dp] * 6 + [_up, _dp] + [_dp] * 4
        L.oracle_srbd_step.restype = i
        L.oracle_srbd_step_rho.argtypes = [PP, i, i, d, d, d] + [_dp] * 6 + [_up, _dp] + [_dp] * 4
        L.oracle_srbd_step_rho.restype = i
        L.oracle_srbd_step_batch.argtypes = [PP, i, i, i, d, d] + [_dp] * 6 + [_up, _dp, _dp, i]
        L.oracle_srbd_plant.argtypes = [PP, _dp, _dp, _dp, _up, C.c_void_p, d, i, _dp]
        MP = C.POINTER(MultiParams)
        L.oracle_multi_coll_cost.argtypes = [MP, _dp]
        L.oracle_multi_coll_cost.restype = d
        L.oracle_multi_linearize.argtypes = [PP, MP, i] + [_dp] * 6 + [_up, _dp] + [_dp] * 11
        L.oracle_multi_linearize.restype = i
        L.oracle_multi_cost.argtypes = [PP, MP, i, _dp, _dp, _dp, _dp, _up]
        L.oracle_multi_cost.restype = d
        L.oracle_multi_theta.argtypes = [PP, MP, i, _dp, _dp, _dp, _up, _dp]
        L.oracle_multi_theta.restype = d
        L.oracle_multi_cost_slope.argtypes = [PP, MP, i, _dp, _dp, _dp, _dp, _up, _dp, _dp]
        L.oracle_multi_cost_slope.restype = d
        L.oracle_multi_step.argtypes = [PP, MP, i, i, d, d] + [_dp] * 6 + [_up, _dp] + [_dp] * 4
        L.oracle_multi_step.restype = i
        L.oracle_max_threads.restype = i
        _lib = L
    return _lib


def _c(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


def max_threads() -> int:
    return lib().oracle_max_threads()


# ----------------------------------------------------------------------------- LQ

def solve_lq_single(qp: dict, b: int = 0):
    """One instance b of a batched LQ dict -> dict with K, k, P, p, dx, du, dlam, info."""
    A = _c(qp["A"][b]); N1, n, _ = A.shape
    N = N1 - 1
    m = qp["Bm"].shape[-1]
    out = {"K": np.zeros((N + 1, m, n)), "k": np.zeros((N + 1, m)), "P": np.zeros((N + 2, n, n)),
           "p": np.zeros((N + 2, n)), "dx": np.zeros((N + 2, n)), "du": np.zeros((N + 1, m)),
           "dlam": np.zeros((N + 2, n))}
    info = lib().oracle_solve_lq(N, n, m, A, _c(qp["Bm"][b]), _c(qp["c"][b]), _c(qp["Q"][b]),
                                 _c(qp["R"][b]), _c(qp["S"][b]), _c(qp["q"][b]), _c(qp["r"][b]),
                                 _c(qp["P_term"][b]), _c(qp["p_term"][b]), _c(qp["dx0"][b]),
                                 out["dx"], out["du"], out["dlam"], out["K"], out["k"], out["P"], out["p"])
    out["info"] = info
    return out


def solve_lq(qp: dict, nthreads: int | None = None):
    """Batched LQ solve -> dict dx[B][N+2][n], du[B][N+1][m], dlam[B][N+2][n], info[B]."""
    A = _c(qp["A"]); Bn, N1, n, _ = A.shape
    m = qp["Bm"].shape[-1]
    N = N1 - 1
    dx = np.zeros((Bn, N + 2, n)); du = np.zeros((Bn, N + 1, m)); dl = np.zeros((Bn, N + 2, n))
    info = np.zeros(Bn, np.int32)
    lib().oracle_solve_lq_batch(Bn, N, n, m, A, _c(qp["Bm"]), _c(qp["c"]), _c(qp["Q"]), _c(qp["R"]),
                                _c(qp["S"]), _c(qp["q"]), _c(qp["r"]), _c(qp["P_term"]),
                                _c(qp["p_term"]), _c(qp["dx0"]), dx, du, dl, info,
                                nthreads or max_threads())
    return {"dx": dx, "du": du, "dlam": dl, "info": info}


def solve_lq_adjoint_single(qp: dict, sol: dict, g: dict, b: int = 0):
    """Gradients of L (dL/d(dx, du, dlam) = g) w.r.t. instance b's Eq. 4 data, given its forward
    solution sol (dict dx, du, dlam of that instance).  Returns (dict of gradients, info)."""
    A = _c(qp["A"][b]); N1, n, _ = A.shape
    N = N1 - 1
    m = qp["Bm"].shape[-1]
    out = {k: np.zeros_like(_c(qp[k][b])) for k in ("A", "Bm", "c", "Q", "R", "S", "q", "r", "P_term", "p_term", "dx0")}
    gz = lambda k, shp: _c(g[k]) if g.get(k) is not None else np.zeros(shp)
    info = lib().oracle_solve_lq_adjoint(
        N, n, m, A, _c(qp["Bm"][b]), _c(qp["Q"][b]), _c(qp["R"][b]), _c(qp["S"][b]), _c(qp["P_term"][b]),
        _c(sol["dx"]), _c(sol["du"]), _c(sol["dlam"]),
        gz("dx", (N + 2, n)), gz("du", (N + 1, m)), gz("dlam", (N + 2, n)),
        out["A"], out["Bm"], out["c"], out["Q"], out["R"], out["S"], out["q"], out["r"], out["P_term"],
        out["p_term"], out["dx0"])
    return out, info


# ----------------------------------------------------------------------------- SRBD

def srbd_f(params: dict, x, u, feet, contact):
    out = np.zeros(12)
    lib().oracle_srbd_f(C.byref(SrbdParams.from_dict(params)), _c(x), _c(u), _c(feet), _c(contact, np.uint8), out)
    return out


def srbd_h(params: dict, x, u, feet, contact):
    out = np.zeros(12)
    lib().oracle_srbd_h(C.byref(SrbdParams.from_dict(params)), _c(x), _c(u), _c(feet), _c(contact, np.uint8), out)
    return out


def srbd_jac(params: dict, x, u, feet, contact):
    Fx = np.zeros((12, 12)); Fu = np.zeros((12, 12))
    lib().oracle_srbd_jac(C.byref(SrbdParams.from_dict(params)), _c(x), _c(u), _c(feet),
                          _c(contact, np.uint8), Fx, Fu)
    return Fx, Fu


def barrier(xi, mu, delta):
    return lib().oracle_barrier(float(xi), float(mu), float(delta))


def barrier_d1(xi, mu, delta):
    return lib().oracle_barrier_d1(float(xi), float(mu), float(delta))


def barrier_d2(xi, mu, delta):
    return lib().oracle_barrier_d2(float(xi), float(mu), float(delta))


def _uref(prob, b=None):
    u = prob.get("u_ref")
    if u is None:
        u = np.zeros_like(prob["u"])
    return _c(u if b is None else u[b])


def srbd_linearize(prob: dict, nthreads: int | None = None):
    """Batched linearisation of an SRBD problem dict (workloads.synth.srbd_problem layout)."""
    x = _c(prob["x"]); Bn, N2, n = x.shape
    N = N2 - 2
    m = 12
    out = {"A": np.zeros((Bn, N + 1, n, n)), "Bm": np.zeros((Bn, N + 1, n, m)), "c": np.zeros((Bn, N + 1, n)),
           "Q": np.zeros((Bn, N + 1, n, n)), "R": np.zeros((Bn, N + 1, m, m)), "S": np.zeros((Bn, N + 1, m, n)),
           "q": np.zeros((Bn, N + 1, n)), "r": np.zeros((Bn, N + 1, m)), "P_term": np.zeros((Bn, n, n)),
           "p_term": np.zeros((Bn, n)), "dx0": np.zeros((Bn, n))}
    info = np.zeros(Bn, np.int32)
    lib().oracle_srbd_linearize_batch(
        C.byref(SrbdParams.from_dict(prob["params"])), Bn, N, x, _c(prob["u"]), _c(prob["lam"]),
        _c(prob["x0"]), _c(prob["x_ref"]), _uref(prob), _c(prob["contact"], np.uint8), _c(prob["feet"]),
        out["A"], out["Bm"], out["c"], out["Q"], out["R"], out["S"], out["q"], out["r"],
        out["P_term"], out["p_term"], out["dx0"], info, nthreads or max_threads())
    out["info"] = info
    return out


def srbd_cost(prob, b, x=None, u=None):
    x = prob["x"][b] if x is None else x
    u = prob["u"][b] if u is None else u
    N = x.shape[0] - 2
    return lib().oracle_srbd_cost(C.byref(SrbdParams.from_dict(prob["params"])), N, _c(x), _c(u),
                                  _c(prob["x_ref"][b]), _uref(prob, b), _c(prob["contact"][b], np.uint8))


def srbd_theta(prob, b, x=None, u=None):
    x = prob["x"][b] if x is None else x
    u = prob["u"][b] if u is None else u
    N = x.shape[0] - 2
    return lib().oracle_srbd_theta(C.byref(SrbdParams.from_dict(prob["params"])), N, _c(x), _c(u),
                                   _c(prob["x0"][b]), _c(prob["contact"][b], np.uint8), _c(prob["feet"][b]))


def srbd_line_search(prob, b, dx, du, n_alpha=10, c1=1e-4, theta_max=None):
    """Returns (j, J[n_alpha], theta[n_alpha], (J0, theta0, slope))."""
    x = prob["x"][b]
    N = x.shape[0] - 2
    tm = 1e-2 * (N + 1) if theta_max is None else theta_max
    Ja = np.zeros(n_alpha); tha = np.zeros(n_alpha); base = np.zeros(3)
    j = lib().oracle_srbd_line_search(C.byref(SrbdParams.from_dict(prob["params"])), N, n_alpha, c1, tm,
                                      _c(x), _c(prob["u"][b]), _c(prob["x0"][b]), _c(prob["x_ref"][b]),
                                      _uref(prob, b), _c(prob["contact"][b], np.uint8), _c(prob["feet"][b]),
                                      _c(dx), _c(du), Ja, tha, base)
    return j, Ja, tha, base


def srbd_step_single(prob, b, n_alpha=10, c1=1e-4, theta_max=0.0, rho=0.0):
    """One SQP iteration of instance b (rho: LM shift added to every R_i, reading R28); returns
    (x, u, lam, stats[5], dx, du, dlam) (copies)."""
    x = _c(prob["x"][b]).copy(); u = _c(prob["u"][b]).copy(); lam = _c(prob["lam"][b]).copy()
    N = x.shape[0] - 2
    st = np.zeros(5)
    dx = np.zeros((N + 2, 12)); du = np.zeros((N + 1, 12)); dl = np.zeros((N + 2, 12))
    lib().oracle_srbd_step_rho(C.byref(SrbdParams.from_dict(prob["params"])), N, n_alpha, c1, theta_max, float(rho),
                               x, u, lam, _c(prob["x0"][b]), _c(prob["x_ref"][b]), _uref(prob, b),
                               _c(prob["contact"][b], np.uint8), _c(prob["feet"][b]), st, dx, du, dl)
    return x, u, lam, st, dx, du, dl


def srbd_step(prob: dict, n_alpha=10, c1=1e-4, theta_max=0.0, nthreads: int | None = None):
    """Batched SRBD step, in place on prob['x'], prob['u'], prob['lam'] (must be float64
    C-contiguous).  Returns stats[B][5] = (cost, theta, alpha, accepted, info)."""
    x = prob["x"]; Bn, N2, _ = x.shape
    N = N2 - 2
    for k in ("x", "u", "lam"):
        assert prob[k].dtype == np.float64 and prob[k].flags.c_contiguous
    st = np.zeros((Bn, 5))
    lib().oracle_srbd_step_batch(C.byref(SrbdParams.from_dict(prob["params"])), Bn, N, n_alpha, c1,
                                 theta_max, prob["x"], prob["u"], prob["lam"], _c(prob["x0"]),
                                 _c(prob["x_ref"]), _uref(prob), _c(prob["contact"], np.uint8),
                                 _c(prob["feet"]), st, nthreads or max_threads())
    return st


def srbd_plant(params: dict, x, u, feet, contact, F_ext=None, dt=0.02, substeps=4):
    """One closed-loop plant step (RK4 of the SRBD dynamics + external CoM force)."""
    out = np.zeros(12)
    fe = None if F_ext is None else _c(F_ext)
    lib().oracle_srbd_plant(C.byref(SrbdParams.from_dict(params)), _c(x), _c(u), _c(feet),
                            _c(contact, np.uint8), None if fe is None else fe.ctypes.data,
                            float(dt), int(substeps), out)
    return out


def warm_start_shift(a):
    """SPEC S:343-350 / P:315: a_i <- a_{i+1} along the stage axis (axis -2), last entry kept."""
    out = np.array(a, copy=True)
    out[..., :-1, :] = a[..., 1:, :]
    return out


def closed_loop(prob_long: dict, N: int, ticks: int, nodes_per_tick: int = 1, substeps: int = 4, push=None,
                n_alpha=10, c1=1e-4, theta_max=0.0):
    """Closed-loop RTI on the oracle.  Each control tick: x0 <- plant state,
    one SQP iteration; then for each of the k = nodes_per_tick nodes until the next tick: the RK4
    plant integrates one node (dt, `substeps` steps) under the plan's first control u_0 with the
    node's contacts/footholds, the iterate is shifted by one node and the reference window slides
    by one node (k = 1: 50 Hz; k = 2: 25 Hz on the same 20 ms nodes, plan played back between
    ticks).  prob_long holds references for >= N + k*ticks stages.  push(node) -> F_ext[B][3] or
    None.  Returns {"x_plant": [B][k*ticks+1][12] (per node), "stats": [B][ticks][5]}."""
    prm = prob_long["params"]
    k = int(nodes_per_tick)
    B = prob_long["x0"].shape[0]
    win = lambda a, o, L: np.ascontiguousarray(a[:, o:o + L])
    it = {"params": prm, "x": win(prob_long["x"], 0, N + 2), "u": win(prob_long["u"], 0, N + 1),
          "lam": win(prob_long["lam"], 0, N + 2)}
    xp = np.array(prob_long["x0"], dtype=np.float64)
    xs, sts = [xp.copy()], []

    def slide(o):
        it.update(x_ref=win(prob_long["x_ref"], o, N + 2), u_ref=win(prob_long["u_ref"], o, N + 1),
                  contact=win(prob_long["contact"], o, N + 1), feet=win(prob_long["feet"], o, N + 1))

    slide(0)
    node = 0
    for t in range(ticks):
        it["x0"] = xp.copy()
        sts.append(srbd_step(it, n_alpha, c1, theta_max))
        for _ in range(k):
            F = push(node) if push is not None else None
            for b in range(B):
                xp[b] = srbd_plant(prm, xp[b], it["u"][b, 0], it["feet"][b, 0], it["contact"][b, 0],
                                   None if F is None else F[b], prm["dt"], substeps)
            for key in ("x", "u", "lam"):
                it[key] = np.ascontiguousarray(warm_start_shift(it[key]))
            node += 1
            slide(node)
            xs.append(xp.copy())
    return {"x_plant": np.stack(xs, 1), "stats": np.stack(sts, 1)}


def srbd_solve(prob: dict, max_iters: int, tol: float, n_alpha=10, c1=1e-4, theta_max=0.0, return_rho=False):
    """Multi-iteration solve, per instance: repeat the SQP iteration until the
    accepted step has theta <= tol and ||alpha (dx, du)||_inf <= tol, or every alpha is rejected at
    a fixed point (theta <= tol and |grad J . (dx, du)| <= tol max(1, |J|), R24)
    (converged at k), or the iteration fails (info < 0, or info > 0 with the LM ladder exhausted:
    stopped, -k), or max_iters.  Levenberg-Marquardt ladder (reading R28): after
    a factorisation failure (info > 0) or an all-rejected search away from a fixed point, the next
    iteration adds rho = 1e-6, then x10 per retry up to 1e-2, to every R_i; an accepted step resets
    rho to 0.  In place on prob x/u/lam.  Returns (iters[B], stats[B][5] of each instance's last
    iteration) (+ final rho[B] if return_rho)."""
    Bn = prob["x"].shape[0]
    iters = np.zeros(Bn, np.int32)
    st = np.zeros((Bn, 5))
    rhos = np.zeros(Bn)
    for b in range(Bn):
        rho = 0.0
        for k in range(1, max_iters + 1):
            x, u, lam, s, dx, du, _ = srbd_step_single(prob, b, n_alpha, c1, theta_max, rho)
            fixed = False
            if s[4] == 0 and not s[3]:
                _, _, _, (J0, th0, g) = srbd_line_search(prob, b, dx, du, n_alpha, c1,
                                                         None if theta_max <= 0 else theta_max)
                fixed = th0 <= tol and abs(g) <= tol * max(1.0, abs(J0))
            prob["x"][b], prob["u"][b], prob["lam"][b] = x, u, lam
            st[b] = s
            retry = False
            if s[3]:
                rho = 0.0
            elif (s[4] > 0 or (s[4] == 0 and not fixed)) and rho < 1e-2:
                rho = 1e-6 if rho == 0.0 else min(10.0 * rho, 1e-2)
                retry = True
            if retry:
                continue
            if s[4] != 0:
                iters[b] = -k
                break
            step = s[2] * max(np.abs(dx).max(), np.abs(du).max())
            if (s[1] <= tol and step <= tol) if s[3] else fixed:
                iters[b] = k
                break
        rhos[b] = rho
    return (iters, st, rhos) if return_rho else (iters, st)

def _mp(prob):
    return C.byref(SrbdParams.from_dict(prob["params"])), C.byref(MultiParams.from_dict(prob["multi"]))


def multi_linearize_single(prob: dict, b: int = 0):
    """Eq. 4 blocks of instance b of a multi-robot problem (workloads.synth.multi_srbd_problem)."""
    x = _c(prob["x"][b]); N = x.shape[0] - 2; n = x.shape[1]
    out = {"A": np.zeros((N + 1, n, n)), "Bm": np.zeros((N + 1, n, n)), "c": np.zeros((N + 1, n)),
           "Q": np.zeros((N + 1, n, n)), "R": np.zeros((N + 1, n, n)), "S": np.zeros((N + 1, n, n)),
           "q": np.zeros((N + 1, n)), "r": np.zeros((N + 1, n)), "P_term": np.zeros((n, n)),
           "p_term": np.zeros(n), "dx0": np.zeros(n)}
    P_, M_ = _mp(prob)
    info = lib().oracle_multi_linearize(P_, M_, N, x, _c(prob["u"][b]), _c(prob["lam"][b]), _c(prob["x0"][b]),
                                        _c(prob["x_ref"][b]), _uref(prob, b), _c(prob["contact"][b], np.uint8),
                                        _c(prob["feet"][b]), out["A"], out["Bm"], out["c"], out["Q"], out["R"],
                                        out["S"], out["q"], out["r"], out["P_term"], out["p_term"], out["dx0"])
    out["info"] = info
    return out


def multi_coll_cost(multi: dict, x_node):
    return lib().oracle_multi_coll_cost(C.byref(MultiParams.from_dict(multi)), _c(x_node))


def multi_cost(prob, b, x=None, u=None):
    x = prob["x"][b] if x is None else x
    u = prob["u"][b] if u is None else u
    P_, M_ = _mp(prob)
    return lib().oracle_multi_cost(P_, M_, x.shape[0] - 2, _c(x), _c(u), _c(prob["x_ref"][b]), _uref(prob, b),
                                   _c(prob["contact"][b], np.uint8))


def multi_theta(prob, b, x=None, u=None):
    x = prob["x"][b] if x is None else x
    u = prob["u"][b] if u is None else u
    P_, M_ = _mp(prob)
    return lib().oracle_multi_theta(P_, M_, x.shape[0] - 2, _c(x), _c(u), _c(prob["x0"][b]),
                                    _c(prob["contact"][b], np.uint8), _c(prob["feet"][b]))


def multi_cost_slope(prob, b, dx, du):
    x = prob["x"][b]
    P_, M_ = _mp(prob)
    return lib().oracle_multi_cost_slope(P_, M_, x.shape[0] - 2, _c(x), _c(prob["u"][b]), _c(prob["x_ref"][b]),
                                         _uref(prob, b), _c(prob["contact"][b], np.uint8), _c(dx), _c(du))


def multi_step_single(prob, b, n_alpha=10, c1=1e-4, theta_max=0.0):
    """One SQP iteration of instance b of the centralized OCP: (x, u, lam, stats[5], dx, du, dlam)."""
    x = _c(prob["x"][b]).copy(); u = _c(prob["u"][b]).copy(); lam = _c(prob["lam"][b]).copy()
    N = x.shape[0] - 2; n = x.shape[1]
    st = np.zeros(5)
    dx = np.zeros((N + 2, n)); du = np.zeros((N + 1, n)); dl = np.zeros((N + 2, n))
    P_, M_ = _mp(prob)
    lib().oracle_multi_step(P_, M_, N, n_alpha, c1, theta_max, x, u, lam, _c(prob["x0"][b]), _c(prob["x_ref"][b]),
                            _uref(prob, b), _c(prob["contact"][b], np.uint8), _c(prob["feet"][b]), st, dx, du, dl)
    return x, u, lam, st, dx, du, dl

