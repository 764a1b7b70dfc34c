"""Prototype of the device algorithm (development aid): Householder
tridiagonalization, static-predicated implicit QL eigenvalues, Sturm count,
inverse iteration with a pivoted tridiagonal LU, back-transform, verification.
Mirrors ys_terms.cuh psd_project9_tri statement by statement.
usage: python tools/evd_proto3.py [state] [samples]   (EVD_SAMPLE=1 samples real H_D on the GPU)"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.argv = sys.argv[:3]

TAU = 1e-12
ORTH = 1e-12


def tridiag(M):
    a = M.copy()
    beta = np.zeros(7)
    e = np.zeros(8)
    V = [None] * 7
    for k in range(7):
        x = a[k + 1:, k].copy()
        sig = (x[1:] ** 2).sum()
        nrm = math.sqrt(x[0] ** 2 + sig)
        if nrm == 0.0:
            e[k] = 0.0
            V[k] = np.zeros(8 - k)
            beta[k] = 0.0
            continue
        alpha = -nrm if x[0] >= 0 else nrm
        v = x.copy()
        v[0] = x[0] - alpha
        b = 1.0 / (nrm * nrm - x[0] * alpha)
        S = a[k + 1:, k + 1:]
        p = b * (S @ v)
        K = 0.5 * b * (p @ v)
        w = p - K * v
        a[k + 1:, k + 1:] = S - np.outer(v, w) - np.outer(w, v)
        e[k] = alpha
        V[k] = v
        beta[k] = b
    e[7] = a[8, 7]
    return np.diag(a).copy(), e, V, beta


def tql(d, e):
    d = d.copy()
    ee = np.zeros(9)
    ee[:8] = e
    for l in range(9):
        it = 0
        while True:
            m = 8
            for i in range(7, -1, -1):
                dd = abs(d[i]) + abs(d[i + 1])
                if i >= l and abs(ee[i]) + dd == dd:
                    m = i
            if m == l:
                break
            if it == 40:
                return None
            it += 1
            dl, dl1, el, dm = d[l], d[l + 1], ee[l], d[m]
            g = (dl1 - dl) / (2.0 * el)
            r = math.hypot(g, 1.0)
            g = dm - dl + el / (g + math.copysign(r, g))
            s = c = 1.0
            p = 0.0
            for i in range(7, -1, -1):
                if l <= i < m:
                    f = s * ee[i]
                    b = c * ee[i]
                    r = math.hypot(f, g)
                    ee[i + 1] = r
                    if r == 0.0:
                        s, c = 0.0, 1.0
                    else:
                        s, c = f / r, g / r
                    g = d[i + 1] - p
                    r = (d[i] - g) * s + 2.0 * c * b
                    p = s * r
                    d[i + 1] = g + p
                    g = c * r - b
            d[l] -= p
            ee[l] = g
            ee[m] = 0.0
    return np.sort(d)


def sturm(d, e, x, pivmin):
    cnt = 0
    q = d[0] - x
    if abs(q) < pivmin:
        q = -pivmin
    cnt += q < 0
    for i in range(1, 9):
        q = d[i] - x - e[i - 1] * e[i - 1] / q
        if abs(q) < pivmin:
            q = -pivmin
        cnt += q < 0
    return cnt


ITS = int(os.environ.get('EVD_ITS', '2'))


def inv_iter(d, e, sig, pivmin, its=None):
    its = ITS if its is None else its
    D = d - sig
    DL = e.copy()
    DU = e.copy()
    DU2 = np.zeros(7)
    piv = np.zeros(8, dtype=bool)
    for i in range(8):
        if abs(D[i]) >= abs(DL[i]):
            if D[i] == 0.0:
                D[i] = pivmin
            fact = DL[i] / D[i]
            DL[i] = fact
            D[i + 1] -= fact * DU[i]
        else:
            fact = D[i] / DL[i]
            D[i] = DL[i]
            DL[i] = fact
            temp = DU[i]
            DU[i] = D[i + 1]
            D[i + 1] = temp - fact * D[i + 1]
            if i < 7:
                DU2[i] = DU[i + 1]
                DU[i + 1] = -fact * DU[i + 1]
            piv[i] = True
    if D[8] == 0.0:
        D[8] = pivmin
    y = np.full(9, 1.0 / 3.0)
    for _ in range(its):
        b = y.copy()
        for i in range(8):
            if piv[i]:
                b[i], b[i + 1] = b[i + 1], b[i]
            b[i + 1] -= DL[i] * b[i]
        b[8] /= D[8]
        b[7] = (b[7] - DU[7] * b[8]) / D[7]
        for i in range(6, -1, -1):
            b[i] = (b[i] - DU[i] * b[i + 1] - DU2[i] * b[i + 2]) / D[i]
        y = b / math.sqrt(b @ b)
    return y


def inv_iter_ldl(d, e, sig, pivmin, its=None):
    """Non-pivoted LDL^T of T - sig I (tiny pivots replaced by pivmin)."""
    its = ITS if its is None else its
    q = np.zeros(9)
    l = np.zeros(8)
    q[0] = d[0] - sig
    for i in range(1, 9):
        if abs(q[i - 1]) < pivmin:
            q[i - 1] = pivmin
        l[i - 1] = e[i - 1] / q[i - 1]
        q[i] = d[i] - sig - l[i - 1] * e[i - 1]
    if abs(q[8]) < pivmin:
        q[8] = pivmin
    y = np.full(9, 1.0 / 3.0)
    for _ in range(its):
        z = y.copy()
        for i in range(1, 9):
            z[i] -= l[i - 1] * z[i - 1]
        z /= q
        for i in range(7, -1, -1):
            z[i] -= l[i] * z[i + 1]
        y = z / math.sqrt(z @ z)
    return y


if os.environ.get("EVD_LDL"):
    inv_iter = inv_iter_ldl  # noqa: F811


def back(V, beta, y):
    x = y.copy()
    for k in range(6, -1, -1):
        s = beta[k] * (V[k] @ x[k + 1:])
        x[k + 1:] -= s * V[k]
    return x


def project(M):
    nrm2 = (M * M).sum()
    nrm = math.sqrt(nrm2)
    d, e, V, beta = tridiag(M)
    lam = tql(d, e)
    if lam is None:
        return None, "ql"
    tn = np.abs(d).max() + 2 * np.abs(e).max()
    pivmin = 1e-300 + 2.2e-16 * tn * 1e-3
    kneg = int((lam < 0).sum())
    if sturm(d, e, 0.0, pivmin) != kneg:
        return None, "sturm"
    if kneg == 0:
        return M.copy(), "pd"
    if kneg <= 3:
        use = list(range(kneg))
    elif 9 - kneg <= 3:
        use = list(range(kneg, 9))
    else:
        return None, "many"
    X = []
    for j in use:
        gap = min(abs(lam[j] - lam[i]) for i in range(9) if i != j)
        if gap <= 1e-10 * nrm:
            return None, "cluster"
        y = inv_iter(d, e, lam[j], pivmin)
        x = back(V, beta, y)
        r = M @ x - lam[j] * x
        if r @ r > TAU * TAU * nrm2:
            return None, "residual"
        for xo in X:
            if abs(xo @ x) > ORTH:
                return None, "orth"
        X.append(x)
    if kneg <= 3:
        P = M.copy()
        for j, x in zip(use, X):
            P -= lam[j] * np.outer(x, x)
    else:
        P = np.zeros_like(M)
        for j, x in zip(use, X):
            P += lam[j] * np.outer(x, x)
    return P, "ok"


def exact(M):
    l, V = np.linalg.eigh(M)
    return (V * np.maximum(l, 0)) @ V.T


def run(mats, label):
    res, err = {}, 0.0
    for M in mats:
        P, why = project(M)
        res[why] = res.get(why, 0) + 1
        if P is not None:
            Pe = exact(M)
            den = np.abs(M).max()
            err = max(err, np.abs(P - Pe).max() / den)
    print(f"{label}: {res} max rel err {err:.2e}", flush=True)


if __name__ == "__main__":
    rng = np.random.default_rng(5)
    rand = []
    for t in range(3000):
        Q = np.linalg.qr(rng.standard_normal((9, 9)))[0]
        l = rng.standard_normal(9) * (10.0 ** rng.uniform(-3, 3))
        if t % 3 == 0:
            l[:3] = l[0] + 1e-9 * rng.standard_normal(3)
        if t % 5 == 0:
            l[4] = 0.0
        M = (Q * l) @ Q.T
        rand.append(0.5 * (M + M.T))
    run(rand, "random")
    if os.environ.get("EVD_SAMPLE"):
        import evd_proto as P0
        run([m for m, _ in P0.HD], "sampled H_D")
