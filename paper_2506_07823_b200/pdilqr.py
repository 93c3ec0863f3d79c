"""Thin Python binding of libpdilqr.so (include/pdilqr.h).  Argument marshalling only: every step
of the hot path runs in the library's CUDA kernels.  PyTorch provides device memory (the
workspace and all arrays are torch tensors), the CUDA stream and process groups.

There is no CPU fallback: if the shared library is missing or fails to load, every entry point
raises.  Names follow include/pdilqr.h.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from . import build as _build

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpdilqr.so")

PDILQR_F32, PDILQR_F64 = 0, 1
PDILQR_MODEL_LQ, PDILQR_MODEL_SRBD, PDILQR_MODEL_MULTI_SRBD = 0, 1, 2
ABI_VERSION = 2
STATUS = {0: "PDILQR_OK", 1: "PDILQR_ERR_INVALID_ARG", 2: "PDILQR_ERR_DIM", 3: "PDILQR_ERR_WORKSPACE",
          4: "PDILQR_ERR_CUDA", 5: "PDILQR_ERR_UNSUPPORTED"}

EXPORTED = ("pdilqr_workspace_bytes", "pdilqr_create", "pdilqr_destroy", "pdilqr_solve_lq",
            "pdilqr_linearize", "pdilqr_step", "pdilqr_tick_host", "pdilqr_last_launch_count",
            "pdilqr_last_error", "pdilqr_abi_version", "pdilqr_profile", "pdilqr_profile_read",
            "pdilqr_shift", "pdilqr_srbd_plant", "pdilqr_solve", "pdilqr_solve_lq_adjoint", "pdilqr_debug_tc_gemm",
            "pdilqr_lq_segment_reduce", "pdilqr_lq_segment_suffix", "pdilqr_lq_segment_forward",
            "pdilqr_lq_segment_prefix")


class SrbdParams(C.Structure):
    _fields_ = [("dt", C.c_double), ("mass", C.c_double), ("inertia", C.c_double * 9),
                ("gravity", C.c_double * 3), ("w_x", C.c_double * 12), ("w_x_term", C.c_double * 12),
                ("w_u_stance", C.c_double), ("w_u_swing", C.c_double), ("mu_friction", C.c_double),
                ("f_min", C.c_double), ("f_max", C.c_double), ("barrier_mu", C.c_double),
                ("barrier_delta", C.c_double)]


class MultiParams(C.Structure):
    _fields_ = [("n_robots", C.c_int32), ("d_min", C.c_double), ("weight", C.c_double), ("sharpness", C.c_double)]


class Config(C.Structure):
    _fields_ = [("N", C.c_int32), ("n", C.c_int32), ("m", C.c_int32), ("batch", C.c_int32),
                ("dtype", C.c_int), ("model", C.c_int), ("n_alpha", C.c_int32), ("armijo_c1", C.c_double),
                ("theta_max", C.c_double), ("leaf_chunk", C.c_int32), ("export_policy", C.c_int32),
                ("srbd", SrbdParams), ("multi", MultiParams)]


class Lq(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("A", "Bm", "c", "Q", "R", "S", "q", "r", "P_term", "p_term", "dx0")]


class Dir(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("dx", "du", "dlam", "K", "k")]


class Iterate(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")]


class Stats(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("cost", "theta", "alpha", "accepted", "info")]


_lib = None


def lib():
    """Load libpdilqr.so (building it first if sources are newer).  Raises if unavailable."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or _build.needs_build():
            _build.build()
        L = C.CDLL(LIB_PATH)
        vp, i32, st = C.c_void_p, C.c_int32, C.c_int
        L.pdilqr_workspace_bytes.argtypes = [C.POINTER(Config), C.POINTER(C.c_size_t)]
        L.pdilqr_create.argtypes = [C.POINTER(Config), C.c_int, vp, C.c_size_t, C.POINTER(vp)]
        L.pdilqr_destroy.argtypes = [vp]
        L.pdilqr_solve_lq.argtypes = [vp, C.POINTER(Lq), C.POINTER(Dir), vp, vp]
        L.pdilqr_solve_lq_adjoint.argtypes = [vp, C.POINTER(Lq), C.POINTER(Dir), C.POINTER(Dir), C.POINTER(Lq), vp, vp]
        L.pdilqr_solve_lq_adjoint.restype = st
        L.pdilqr_debug_tc_gemm.argtypes = [i32, i32, i32, i32, i32, vp, i32, vp, i32, vp, vp, vp]
        L.pdilqr_debug_tc_gemm.restype = st
        L.pdilqr_lq_segment_reduce.argtypes = [vp, C.POINTER(Lq), vp, vp, vp]
        L.pdilqr_lq_segment_suffix.argtypes = [vp, vp, i32, i32, vp, vp, vp, vp, vp]
        L.pdilqr_lq_segment_forward.argtypes = [vp, C.POINTER(Lq), vp, vp]
        L.pdilqr_lq_segment_prefix.argtypes = [vp, vp, i32, i32, vp, vp, vp]
        for f in ("pdilqr_lq_segment_reduce", "pdilqr_lq_segment_suffix", "pdilqr_lq_segment_forward",
                  "pdilqr_lq_segment_prefix"):
            getattr(L, f).restype = st
        L.pdilqr_linearize.argtypes = [vp, C.POINTER(Iterate), C.POINTER(Lq), vp, vp]
        L.pdilqr_step.argtypes = [vp, C.POINTER(Iterate), C.POINTER(Stats), C.POINTER(Dir), vp]
        L.pdilqr_tick_host.argtypes = [vp, C.POINTER(Iterate), vp, vp, vp, vp, vp, vp, vp, vp]
        L.pdilqr_last_launch_count.argtypes = [vp]
        L.pdilqr_last_launch_count.restype = i32
        L.pdilqr_last_error.restype = C.c_char_p
        L.pdilqr_abi_version.restype = i32
        L.pdilqr_profile.argtypes = [vp, i32]
        L.pdilqr_profile.restype = st
        L.pdilqr_profile_read.argtypes = [vp, i32, C.POINTER(C.c_char_p), C.POINTER(i32), C.POINTER(C.c_double)]
        L.pdilqr_profile_read.restype = i32
        L.pdilqr_solve.argtypes = [vp, C.POINTER(Iterate), i32, C.c_double, C.POINTER(Stats), vp,
                                   C.POINTER(C.c_int32), vp]
        L.pdilqr_solve.restype = st
        L.pdilqr_shift.argtypes = [vp, C.POINTER(Iterate), vp]
        L.pdilqr_shift.restype = st
        L.pdilqr_srbd_plant.argtypes = [vp, C.POINTER(Iterate), vp, vp, vp, C.c_double, i32, vp]
        L.pdilqr_srbd_plant.restype = st
        for f in ("pdilqr_workspace_bytes", "pdilqr_create", "pdilqr_destroy", "pdilqr_solve_lq",
                  "pdilqr_linearize", "pdilqr_step", "pdilqr_tick_host"):
            getattr(L, f).restype = st
        _lib = L
    return _lib


class PdilqrError(RuntimeError):
    pass


def debug_tc_gemm(A, B, Cin=None, trans_a=False, trans_b=False, stream=None):
    """pdilqr_debug_tc_gemm: C = Cin + op(A) op(B) through the tcgen05 3xTF32 product of the large-n
    fold (one CTA; diagnostic).  float32 CUDA tensors, row-major."""
    M = A.shape[1] if trans_a else A.shape[0]
    K = A.shape[0] if trans_a else A.shape[1]
    N = B.shape[0] if trans_b else B.shape[1]
    for t in (A, B) + ((Cin,) if Cin is not None else ()):
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
            raise PdilqrError("debug_tc_gemm: contiguous float32 CUDA tensors expected")
    C = torch.empty(M, N, dtype=torch.float32, device=A.device)
    s = torch.cuda.current_stream(A.device) if stream is None else stream
    _check(lib().pdilqr_debug_tc_gemm(M, N, K, int(trans_a), int(trans_b), _ptr(A), A.shape[1], _ptr(B), B.shape[1],
                                      _ptr(Cin), _ptr(C), C_void(s.cuda_stream)))
    return C


def C_void(x):
    return C.c_void_p(x)


def _check(status: int):
    if status != 0:
        raise PdilqrError(f"{STATUS.get(status, status)}: {lib().pdilqr_last_error().decode()}")


def srbd_params_struct(d: dict | None) -> SrbdParams:
    p = SrbdParams()
    if d is None:
        return p
    for name, _ in SrbdParams._fields_:
        v = d[name]
        if isinstance(v, (list, tuple)):
            arr = getattr(p, name)
            for i, e in enumerate(v):
                arr[i] = float(e)
        else:
            setattr(p, name, float(v))
    return p


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


class PdIlqr:
    """One library handle: fixed (N, n, m, batch, dtype, model) on one CUDA device.

    The workspace is a torch uint8 tensor owned by this object.  All array arguments must be
    contiguous CUDA tensors of the handle's dtype (contact: uint8) on the handle's device.
    """

    def __init__(self, N: int, n: int, m: int, batch: int, dtype=torch.float32, model: str = "lq",
                 srbd: dict | None = None, n_alpha: int = 10, armijo_c1: float = 1e-4, theta_max: float = 0.0,
                 leaf_chunk: int = 0, device: int | torch.device | None = None, multi: dict | None = None):
        L = lib()
        if L.pdilqr_abi_version() != ABI_VERSION:
            raise PdilqrError(f"libpdilqr.so ABI {L.pdilqr_abi_version()} != binding ABI {ABI_VERSION}")
        self.N, self.n, self.m, self.batch = N, n, m, batch
        self.dtype = dtype
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   (device.index if isinstance(device, torch.device) else device))
        mdl = {"lq": PDILQR_MODEL_LQ, "srbd": PDILQR_MODEL_SRBD, "multi_srbd": PDILQR_MODEL_MULTI_SRBD}[model]
        mp = MultiParams(**({k: multi[k] for k in ("n_robots", "d_min", "weight", "sharpness")} if multi else {}))
        cfg = Config(N=N, n=n, m=m, batch=batch, dtype=PDILQR_F32 if dtype == torch.float32 else PDILQR_F64,
                     model=mdl, n_alpha=n_alpha, armijo_c1=armijo_c1, theta_max=theta_max, leaf_chunk=leaf_chunk,
                     export_policy=0, srbd=srbd_params_struct(srbd), multi=mp)
        self.model = model
        self.n_robots = multi["n_robots"] if multi else 1
        self._cfg = cfg
        nb = C.c_size_t()
        _check(L.pdilqr_workspace_bytes(C.byref(cfg), C.byref(nb)))
        self.workspace = torch.empty(max(nb.value, 256), dtype=torch.uint8, device=self.device)
        h = C.c_void_p()
        _check(L.pdilqr_create(C.byref(cfg), self.device.index, C.c_void_p(self.workspace.data_ptr()),
                               nb.value, C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.pdilqr_destroy(h)
            self._h = None

    # ------------------------------------------------------------------ helpers
    def _check_t(self, t, shape, dtype=None):
        dtype = dtype or self.dtype
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dtype and t.is_contiguous()
                and t.device == self.device and tuple(t.shape) == tuple(shape)):
            raise PdilqrError(f"expected contiguous {dtype} tensor of shape {tuple(shape)} on {self.device}, "
                              f"got {getattr(t, 'dtype', type(t))} {tuple(getattr(t, 'shape', ()))} "
                              f"on {getattr(t, 'device', None)}")
        return t

    def _check_host(self, t, shape, dtype=None):
        dtype = dtype or self.dtype
        if not (isinstance(t, torch.Tensor) and t.device.type == "cpu" and t.dtype == dtype and t.is_contiguous()
                and tuple(t.shape) == tuple(shape)):
            raise PdilqrError(f"expected contiguous host {dtype} tensor of shape {tuple(shape)}, got "
                              f"{getattr(t, 'dtype', type(t))} {tuple(getattr(t, 'shape', ()))} "
                              f"on {getattr(t, 'device', None)}")
        if not t.is_pinned():
            raise PdilqrError("host buffers of tick_host must be pinned (asynchronous copies)")
        return t

    def _check_dir(self, d: dict, policy_ok: bool = True):
        B, N, n, m = self.batch, self.N, self.n, self.m
        self._check_t(d["dx"], (B, N + 2, n)); self._check_t(d["du"], (B, N + 1, m))
        self._check_t(d["dlam"], (B, N + 2, n))
        if d.get("K") is not None:
            self._check_t(d["K"], (B, N + 1, m, n))
        if d.get("k") is not None:
            self._check_t(d["k"], (B, N + 1, m))
        return d

    def _stream(self, stream):
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        return C.c_void_p(s.cuda_stream)

    def lq_shapes(self):
        B, N, n, m = self.batch, self.N, self.n, self.m
        return {"A": (B, N + 1, n, n), "Bm": (B, N + 1, n, m), "c": (B, N + 1, n), "Q": (B, N + 1, n, n),
                "R": (B, N + 1, m, m), "S": (B, N + 1, m, n), "q": (B, N + 1, n), "r": (B, N + 1, m),
                "P_term": (B, n, n), "p_term": (B, n), "dx0": (B, n)}

    def new_direction(self, policy: bool = False):
        B, N, n, m = self.batch, self.N, self.n, self.m
        kw = dict(dtype=self.dtype, device=self.device)
        d = {"dx": torch.empty(B, N + 2, n, **kw), "du": torch.empty(B, N + 1, m, **kw),
             "dlam": torch.empty(B, N + 2, n, **kw)}
        if policy:
            d["K"] = torch.empty(B, N + 1, m, n, **kw)
            d["k"] = torch.empty(B, N + 1, m, **kw)
        return d

    # ------------------------------------------------------------------ entry points
    def solve_lq(self, qp: dict, out: dict | None = None, policy: bool = False, info=None, stream=None):
        """pdilqr_solve_lq: returns dict dx, du, dlam (+ K, k) and info (int32 [B])."""
        for k, shp in self.lq_shapes().items():
            self._check_t(qp[k], shp)
        out = self._check_dir(out) if out is not None else self.new_direction(policy)
        info = self._check_t(info, (self.batch,), torch.int32) if info is not None else \
            torch.empty(self.batch, dtype=torch.int32, device=self.device)
        lq = Lq(**{k: _ptr(qp[k]) for k in self.lq_shapes()})
        d = Dir(dx=_ptr(out["dx"]), du=_ptr(out["du"]), dlam=_ptr(out["dlam"]), K=_ptr(out.get("K")),
                k=_ptr(out.get("k")))
        _check(lib().pdilqr_solve_lq(self._h, C.byref(lq), C.byref(d), _ptr(info), self._stream(stream)))
        out["info"] = info
        return out

    def solve_lq_adjoint(self, qp: dict, sol: dict, gsol: dict, grad: dict | None = None, info=None, stream=None):
        """pdilqr_solve_lq_adjoint: gradients of a loss L w.r.t. the Eq. 4 data, given the forward
        solution sol (dx, du, dlam) of the same qp and gsol = dL/d(dx, du, dlam) (missing keys = 0).
        Returns dict of gradient tensors (the keys of grad, default all 11) and info."""
        shapes = self.lq_shapes()
        for k in ("A", "Bm", "Q", "R", "S", "P_term"):
            self._check_t(qp[k], shapes[k])
        self._check_dir(sol)
        B, N, n, m = self.batch, self.N, self.n, self.m
        gs = {"dx": (B, N + 2, n), "du": (B, N + 1, m), "dlam": (B, N + 2, n)}
        for k, shp in gs.items():
            if gsol.get(k) is not None:
                self._check_t(gsol[k], shp)
        if grad is None:
            grad = {k: torch.empty(shp, dtype=self.dtype, device=self.device) for k, shp in shapes.items()}
        for k, t in grad.items():
            if k != "info":
                self._check_t(t, shapes[k])
        info = self._check_t(info, (B,), torch.int32) if info is not None else \
            torch.empty(B, dtype=torch.int32, device=self.device)
        lq = Lq(**{k: _ptr(qp.get(k)) for k in shapes})
        d = Dir(dx=_ptr(sol["dx"]), du=_ptr(sol["du"]), dlam=_ptr(sol["dlam"]), K=None, k=None)
        g = Dir(dx=_ptr(gsol.get("dx")), du=_ptr(gsol.get("du")), dlam=_ptr(gsol.get("dlam")), K=None, k=None)
        gr = Lq(**{k: _ptr(grad.get(k)) for k in shapes})
        _check(lib().pdilqr_solve_lq_adjoint(self._h, C.byref(lq), C.byref(d), C.byref(g), C.byref(gr), _ptr(info),
                                             self._stream(stream)))
        grad["info"] = info
        return grad

    # ---------------------------------------------------------- horizon sharding (NEXT-2)
    def segment_reduce(self, qp: dict, out=None, info=None, stream=None):
        """pdilqr_lq_segment_reduce: chunk summary S = e_0 (x) ... (x) e_N, [B][3 n^2 + 2 n]."""
        for k, shp in self.lq_shapes().items():
            self._check_t(qp[k], shp)
        B, n = self.batch, self.n
        out = self._check_t(out, (B, 3 * n * n + 2 * n)) if out is not None else \
            torch.empty(B, 3 * n * n + 2 * n, dtype=self.dtype, device=self.device)
        lq = Lq(**{k: _ptr(qp[k]) for k in self.lq_shapes()})
        _check(lib().pdilqr_lq_segment_reduce(self._h, C.byref(lq), _ptr(out), _ptr(info), self._stream(stream)))
        return out

    def segment_suffix(self, S_all, r: int, P_term, p_term, stream=None):
        """pdilqr_lq_segment_suffix: (P, p) of S_{r+1} (x) ... (x) S_{G-1} (x) (P_term, p_term)."""
        B, n = self.batch, self.n
        G = S_all.shape[0]
        self._check_t(S_all, (G, B, 3 * n * n + 2 * n)); self._check_t(P_term, (B, n, n)); self._check_t(p_term, (B, n))
        P = torch.empty(B, n, n, dtype=self.dtype, device=self.device)
        p = torch.empty(B, n, dtype=self.dtype, device=self.device)
        _check(lib().pdilqr_lq_segment_suffix(self._h, _ptr(S_all), G, int(r), _ptr(P_term), _ptr(p_term), _ptr(P),
                                              _ptr(p), self._stream(stream)))
        return P, p

    def segment_forward(self, qp: dict, stream=None):
        """pdilqr_lq_segment_forward: closed-loop map (Phi, phi) of the last solve_lq on qp, [B][n^2 + n]."""
        B, n = self.batch, self.n
        shapes = self.lq_shapes()
        for k in ("A", "Bm", "c"):
            self._check_t(qp[k], shapes[k])
        F = torch.empty(B, n * n + n, dtype=self.dtype, device=self.device)
        lq = Lq(**{k: _ptr(qp.get(k)) for k in shapes})
        _check(lib().pdilqr_lq_segment_forward(self._h, C.byref(lq), _ptr(F), self._stream(stream)))
        return F

    def segment_prefix(self, F_all, r: int, dx0, stream=None):
        """pdilqr_lq_segment_prefix: dx at this rank's first node from the gathered maps and dx0."""
        B, n = self.batch, self.n
        G = F_all.shape[0]
        self._check_t(F_all, (G, B, n * n + n)); self._check_t(dx0, (B, n))
        dxs = torch.empty(B, n, dtype=self.dtype, device=self.device)
        _check(lib().pdilqr_lq_segment_prefix(self._h, _ptr(F_all), G, int(r), _ptr(dx0), _ptr(dxs),
                                              self._stream(stream)))
        return dxs

    def _iterate(self, it: dict) -> Iterate:
        B, N, R = self.batch, self.N, self.n_robots
        nx = 12 * R
        self._check_t(it["x"], (B, N + 2, nx)); self._check_t(it["u"], (B, N + 1, nx))
        self._check_t(it["lam"], (B, N + 2, nx)); self._check_t(it["x0"], (B, nx))
        self._check_t(it["x_ref"], (B, N + 2, nx))
        if it.get("u_ref") is not None:
            self._check_t(it["u_ref"], (B, N + 1, nx))
        self._check_t(it["contact"], (B, N + 1, 4 * R), torch.uint8)
        self._check_t(it["feet"], (B, N + 1, 4 * R, 3))
        return Iterate(**{k: _ptr(it.get(k)) for k in ("x", "u", "lam", "x0", "x_ref", "u_ref", "contact", "feet")})

    def linearize(self, it: dict, out: dict | None = None, info=None, stream=None):
        """pdilqr_linearize: the Eq. 4 data at the iterate (dict of tensors) and info."""
        if out is None:
            out = {k: torch.empty(s, dtype=self.dtype, device=self.device) for k, s in self.lq_shapes().items()}
        info = info if info is not None else torch.empty(self.batch, dtype=torch.int32, device=self.device)
        itc = self._iterate(it)
        lq = Lq(**{k: _ptr(out[k]) for k in self.lq_shapes()})
        _check(lib().pdilqr_linearize(self._h, C.byref(itc), C.byref(lq), _ptr(info), self._stream(stream)))
        out["info"] = info
        return out

    def new_stats(self):
        kw = dict(device=self.device)
        return {"cost": torch.empty(self.batch, dtype=self.dtype, **kw),
                "theta": torch.empty(self.batch, dtype=self.dtype, **kw),
                "alpha": torch.empty(self.batch, dtype=self.dtype, **kw),
                "accepted": torch.empty(self.batch, dtype=torch.int32, **kw),
                "info": torch.empty(self.batch, dtype=torch.int32, **kw)}

    def step(self, it: dict, stats: dict | None = None, direction: dict | None = None, stream=None):
        """pdilqr_step: one SQP/RTI iteration, updates it['x'], it['u'], it['lam'] in place."""
        stats = stats if stats is not None else self.new_stats()
        itc = self._iterate(it)
        st = Stats(**{k: _ptr(stats[k]) for k in ("cost", "theta", "alpha", "accepted", "info")})
        d = None
        if direction is not None:
            self._check_dir(direction)
            d = Dir(dx=_ptr(direction["dx"]), du=_ptr(direction["du"]), dlam=_ptr(direction["dlam"]),
                    K=_ptr(direction.get("K")), k=_ptr(direction.get("k")))
        _check(lib().pdilqr_step(self._h, C.byref(itc), C.byref(st), C.byref(d) if d is not None else None,
                                 self._stream(stream)))
        return stats

    def tick_host(self, it: dict, x0_host, u0_host, stats_host: dict, stream=None):
        """pdilqr_tick_host: host x0 in, host u0 + stats out (pinned CPU tensors)."""
        itc = self._iterate(it)
        B = self.batch
        self._check_host(x0_host, (B, 12)); self._check_host(u0_host, (B, 12))
        for k in ("cost", "theta", "alpha"):
            self._check_host(stats_host[k], (B,))
        for k in ("accepted", "info"):
            self._check_host(stats_host[k], (B,), torch.int32)
        _check(lib().pdilqr_tick_host(self._h, C.byref(itc), _ptr(x0_host), _ptr(u0_host),
                                      _ptr(stats_host["cost"]), _ptr(stats_host["theta"]),
                                      _ptr(stats_host["alpha"]), _ptr(stats_host["accepted"]),
                                      _ptr(stats_host["info"]), self._stream(stream)))

    def capture_tick_host(self, it: dict, x0_host, u0_host, stats_host: dict, warmup: int = 1):
        """pdilqr_tick_host captured once into a CUDA graph (the library call is graph-capturable:
        no allocation, no host sync).  Returns the graph: per control tick the caller writes
        x0_host, calls graph.replay(), synchronises, and reads u0_host / stats_host -- the same
        copies and kernels as tick_host without the per-call host launch work."""
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.tick_host(it, x0_host, u0_host, stats_host, stream=s)
            s.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                self.tick_host(it, x0_host, u0_host, stats_host, stream=s)
        torch.cuda.current_stream(self.device).wait_stream(s)
        return g

    def solve(self, it: dict, max_iters: int = 50, tol: float = 1e-6, stats: dict | None = None, stream=None):
        """pdilqr_solve: SQP iterations until every instance converged (theta <= tol and step <= tol)
        or max_iters.  Returns (stats, iters[B] device int32, iterations run)."""
        stats = stats if stats is not None else self.new_stats()
        itc = self._iterate(it)
        sc = Stats(**{k: _ptr(stats[k]) for k in ("cost", "theta", "alpha", "accepted", "info")})
        iters = torch.empty(self.batch, dtype=torch.int32, device=self.device)
        run = C.c_int32(0)
        _check(lib().pdilqr_solve(self._h, C.byref(itc), int(max_iters), float(tol), C.byref(sc), _ptr(iters),
                                  C.byref(run), self._stream(stream)))
        return stats, iters, run.value

    def shift(self, it: dict, stream=None):
        """pdilqr_shift: warm start for the next tick."""
        itc = self._iterate(it)
        _check(lib().pdilqr_shift(self._h, C.byref(itc), self._stream(stream)))

    def plant(self, it: dict, x_plant, u_hold, ext_force=None, dt: float = 0.02, substeps: int = 4, stream=None):
        """pdilqr_srbd_plant: RK4 SRBD plant step (closed-loop simulation), x_plant updated in place."""
        itc = self._iterate(it)
        self._check_t(x_plant, (self.batch, 12))
        self._check_t(u_hold, (self.batch, 12))
        if ext_force is not None:
            self._check_t(ext_force, (self.batch, 3))
        _check(lib().pdilqr_srbd_plant(self._h, C.byref(itc), _ptr(x_plant), _ptr(u_hold), _ptr(ext_force),
                                       float(dt), int(substeps), self._stream(stream)))

    def profile(self, enable: bool = True):
        """Enable / disable per-kernel CUDA-event timing inside the library."""
        _check(lib().pdilqr_profile(self._h, 1 if enable else 0))

    def profile_read(self) -> dict:
        """{kernel: (launches, total_ms)} since the last read / enable (synchronises)."""
        mx = 32
        names = (C.c_char_p * mx)(); cnt = (C.c_int32 * mx)(); tot = (C.c_double * mx)()
        n = lib().pdilqr_profile_read(self._h, mx, names, cnt, tot)
        return {names[k].decode(): (int(cnt[k]), float(tot[k])) for k in range(min(n, mx))}

    def last_launch_count(self) -> int:
        return int(lib().pdilqr_last_launch_count(self._h))
