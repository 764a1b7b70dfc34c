"""Prototype: Householder tridiagonalization + tridiagonal eigenvalues +
inverse iteration for the clamped eigenpairs only (development aid).
usage: python tools/evd_proto2.py [state] [samples]"""
import os
import sys

import numpy as np
from scipy.linalg import eigh_tridiagonal

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.argv = sys.argv[:3]
import evd_proto as P0  # noqa: E402  (sample_hd)


def householder_tridiag(M):
    A = M.copy()
    n = 9
    refl = []
    for k in range(n - 2):
        x = A[k + 1:, k].copy()
        alpha = -np.copysign(np.linalg.norm(x), x[0]) if x[0] != 0 else -np.linalg.norm(x)
        v = x.copy()
        v[0] -= alpha
        vn2 = v @ v
        if vn2 == 0:
            refl.append((np.zeros_like(v), 0.0))
            continue
        beta = 2.0 / vn2
        refl.append((v, beta))
        S = A[k + 1:, k + 1:]
        p = beta * (S @ v)
        w = p - 0.5 * beta * (p @ v) * v
        A[k + 1:, k + 1:] = S - np.outer(v, w) - np.outer(w, v)
        A[k + 1:, k] = 0
        A[k, k + 1:] = 0
        A[k + 1, k] = A[k, k + 1] = alpha
    d = np.diag(A).copy()
    e = np.diag(A, 1).copy()
    return d, e, refl


def apply_Q(refl, y):
    # Q = H_0 H_1 ... H_6 ; eigenvector of M = Q y
    x = y.copy()
    for k in reversed(range(len(refl))):
        v, beta = refl[k]
        x[k + 1:] -= beta * (v @ x[k + 1:]) * v
    return x


def inv_iter(d, e, lam, nrm, iters=2):
    n = len(d)
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    shift = lam + 1e-14 * nrm  # tiny perturbation keeps T - shift nonsingular
    x = np.ones(n) / 3.0
    for _ in range(iters):
        x = np.linalg.solve(T - shift * np.eye(n), x)
        x /= np.linalg.norm(x)
    return x


def proj_tri(M, clust=1e-6, tol_res=1e-11, delta=1e-11):
    nrm = np.linalg.norm(M)
    d, e, refl = householder_tridiag(M)
    lam = eigh_tridiagonal(d, e, eigvals_only=True)
    neg = np.where(lam < 0)[0]
    if len(neg) == 0:
        return M.copy(), "pd"
    use = neg if len(neg) <= 4 else np.where(lam >= 0)[0]
    # cluster test among the eigenvalues whose vectors we need (and their neighbours)
    for i in use:
        for j in range(9):
            if j != i and abs(lam[i] - lam[j]) < clust * nrm:
                return None, "cluster"
    vecs = [apply_Q(refl, inv_iter(d, e, lam[i], nrm)) for i in use]
    for i, v in zip(use, vecs):
        if np.linalg.norm(M @ v - lam[i] * v) > tol_res * nrm:
            return None, "residual"
    if len(neg) <= 4:
        P = M.copy()
        for i, v in zip(use, vecs):
            P -= lam[i] * np.outer(v, v)
    else:
        P = np.zeros_like(M)
        for i, v in zip(use, vecs):
            P += lam[i] * np.outer(v, v)
    try:
        np.linalg.cholesky(P + delta * nrm * np.eye(9))
    except np.linalg.LinAlgError:
        return None, "psd"
    return P, "ok"


HD = P0.HD
for clust in (1e-3, 1e-5, 1e-7):
    res, err = {}, 0.0
    for M, _ in HD:
        Pm, why = proj_tri(M, clust)
        res[why] = res.get(why, 0) + 1
        if Pm is not None:
            Pe, _ = P0.proj_exact(M)
            err = max(err, np.abs(Pm - Pe).max() / np.abs(Pe).max())
    print(f"cluster {clust:g}: {res} max rel err {err:.2e}", flush=True)
# adversarial: random symmetric with clusters / many negatives
rng = np.random.default_rng(5)
res, err = {}, 0.0
for t in range(3000):
    Q = np.linalg.qr(rng.standard_normal((9, 9)))[0]
    l = rng.standard_normal(9)
    if t % 3 == 0:
        l[:3] = l[0] + 1e-9 * rng.standard_normal(3)
    M = (Q * l) @ Q.T
    M = 0.5 * (M + M.T)
    Pm, why = proj_tri(M, 1e-5)
    res[why] = res.get(why, 0) + 1
    if Pm is not None:
        Pe, _ = P0.proj_exact(M)
        err = max(err, np.abs(Pm - Pe).max() / np.abs(Pe).max())
print(f"random: {res} max rel err {err:.2e}")
