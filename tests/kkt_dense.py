"""Dense KKT assembly of the Eq. 4 QP for tests.

This is the *definition* of the LQ subproblem's solution, written out: the first-order
optimality system of

    min  sum_{i=0}^{N} [q_i; r_i]^T [dx_i; du_i] + 1/2 [dx_i; du_i]^T [[Q_i, S_i^T], [S_i, R_i]] [dx_i; du_i]
         + p_{N+1}^T dx_{N+1} + 1/2 dx_{N+1}^T P_{N+1} dx_{N+1}
    s.t. dx_0 = dx0,  dx_{i+1} = A_i dx_i + B_i du_i + b_i

with multipliers attached as in the paper's Lagrangian (sign of SPEC S:120):
    L = f + lam_0^T (dx0 - dx_0) + sum_i lam_{i+1}^T (A_i dx_i + B_i du_i + b_i - dx_{i+1}).
Solved with numpy.linalg.solve (LAPACK LU).  Used to pin the oracle (tests/test_oracle_lq.py) and
to compute KKT backward errors of GPU outputs blockwise in fp64 (tests/test_gpu_*.py).
"""
import numpy as np


def assemble(qp, b=0):
    A, Bm, c = qp["A"][b], qp["Bm"][b], qp["c"][b]
    Q, R, S, q, r = qp["Q"][b], qp["R"][b], qp["S"][b], qp["q"][b], qp["r"][b]
    Pt, pt, dx0 = qp["P_term"][b], qp["p_term"][b], qp["dx0"][b]
    N = A.shape[0] - 1
    n, m = A.shape[1], Bm.shape[2]
    nz = (N + 2) * n + (N + 1) * m          # primal variables: dx_0..dx_{N+1}, du_0..du_N
    nc = (N + 2) * n                        # constraints: initial condition + N+1 dynamics
    X = lambda i: slice(i * n, (i + 1) * n)
    U = lambda i: slice((N + 2) * n + i * m, (N + 2) * n + (i + 1) * m)
    H = np.zeros((nz, nz)); h = np.zeros(nz)
    J = np.zeros((nc, nz)); g = np.zeros(nc)
    for i in range(N + 1):
        H[X(i), X(i)] += Q[i]; H[U(i), U(i)] += R[i]
        H[U(i), X(i)] += S[i]; H[X(i), U(i)] += S[i].T
        h[X(i)] += q[i]; h[U(i)] += r[i]
    H[X(N + 1), X(N + 1)] += Pt; h[X(N + 1)] += pt
    C = lambda k: slice(k * n, (k + 1) * n)
    J[C(0), X(0)] = -np.eye(n); g[C(0)] = dx0               # dx0 - dx_0 = 0
    for i in range(N + 1):                                   # A dx_i + B du_i + b_i - dx_{i+1} = 0
        J[C(i + 1), X(i)] = A[i]; J[C(i + 1), U(i)] = Bm[i]; J[C(i + 1), X(i + 1)] = -np.eye(n)
        g[C(i + 1)] = c[i]
    # stationarity: H z + h + J^T lam = 0 ; feasibility: J z + g = 0
    M = np.block([[H, J.T], [J, np.zeros((nc, nc))]])
    rhs = np.concatenate([-h, -g])
    return M, rhs, (N, n, m)


def unpack(sol, dims):
    N, n, m = dims
    nx = (N + 2) * n
    dx = sol[:nx].reshape(N + 2, n)
    du = sol[nx:nx + (N + 1) * m].reshape(N + 1, m)
    lam = sol[nx + (N + 1) * m:].reshape(N + 2, n)
    return dx, du, lam


def solve(qp, b=0):
    M, rhs, dims = assemble(qp, b)
    return unpack(np.linalg.solve(M, rhs), dims)


def backward_error(qp, b, dx, du, dlam):
    """Normwise backward error eta = ||M z - rhs||_inf / (||M||_inf ||z||_inf + ||rhs||_inf)
    (SURVEY §8(c-5)), in fp64.  Dense; use for N*(n+m) up to a few thousand."""
    M, rhs, dims = assemble(qp, b)
    z = np.concatenate([np.asarray(dx, np.float64).ravel(), np.asarray(du, np.float64).ravel(),
                        np.asarray(dlam, np.float64).ravel()])
    res = M @ z - rhs
    return np.abs(res).max() / (np.abs(M).sum(axis=1).max() * np.abs(z).max() + np.abs(rhs).max())


def backward_error_blockwise(qp, b, dx, du, dlam):
    """Same eta, computed block by block (no dense M); scales to any N."""
    A, Bm, c = qp["A"][b], qp["Bm"][b], qp["c"][b]
    Q, R, S, q, r = qp["Q"][b], qp["R"][b], qp["S"][b], qp["q"][b], qp["r"][b]
    Pt, pt, dx0 = qp["P_term"][b], qp["p_term"][b], qp["dx0"][b]
    dx = np.asarray(dx, np.float64); du = np.asarray(du, np.float64); dl = np.asarray(dlam, np.float64)
    N = A.shape[0] - 1
    n = A.shape[1]
    res = []; rown = []
    absI = np.ones(n)
    # x-rows: Q dx + S^T du + q + A^T lam_{i+1} - lam_i
    for i in range(N + 1):
        res.append(Q[i] @ dx[i] + S[i].T @ du[i] + q[i] + A[i].T @ dl[i + 1] - dl[i])
        rown.append(np.abs(Q[i]).sum(1) + np.abs(S[i].T).sum(1) + np.abs(A[i].T).sum(1) + absI)
    res.append(Pt @ dx[N + 1] + pt - dl[N + 1])
    rown.append(np.abs(Pt).sum(1) + absI)
    for i in range(N + 1):  # u-rows: S dx + R du + r + B^T lam_{i+1}
        res.append(S[i] @ dx[i] + R[i] @ du[i] + r[i] + Bm[i].T @ dl[i + 1])
        rown.append(np.abs(S[i]).sum(1) + np.abs(R[i]).sum(1) + np.abs(Bm[i].T).sum(1))
    res.append(-dx[0] + dx0); rown.append(absI)
    for i in range(N + 1):
        res.append(A[i] @ dx[i] + Bm[i] @ du[i] + c[i] - dx[i + 1])
        rown.append(np.abs(A[i]).sum(1) + np.abs(Bm[i]).sum(1) + absI)
    rhs_inf = max(np.abs(q).max(), np.abs(r).max(), np.abs(pt).max(), np.abs(dx0).max(), np.abs(c).max())
    z_inf = max(np.abs(dx).max(), np.abs(du).max(), np.abs(dl).max())
    M_inf = max(v.max() for v in rown)
    return max(np.abs(v).max() for v in res) / (M_inf * z_inf + rhs_inf)
