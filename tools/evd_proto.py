"""Prototype of the subspace PSD projection for the SNH 9x9 edge-space Hessian
(development aid): samples H_D of C5 tets at the bench's prepared state, then
compares the inverse-subspace-iteration projection with numpy's eigh.
usage: python tools/evd_proto.py [state] [samples]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

state = sys.argv[1] if len(sys.argv) > 1 else "rollout"
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 20000


def sample_hd():
    from bench import prepare
    from paper_2605_23088_b200.scene import make_tet_block
    sim = prepare("c5", True, "gpu", state=state)
    out = []
    E, nu = 20000.0, 0.3
    mu, lam = E / (2 * (1 + nu)), E * nu / ((1 + nu) * (1 - 2 * nu))
    alpha = 1 + 3 * mu / (4 * lam)
    w = sim.config.dt ** 2
    rng = np.random.default_rng(0)
    for b, bj in zip(sim.bodies, sim.config.bodies):
        if bj.get("kind") != "tet_block":
            continue
        rest, tets = make_tet_block(bj["nx"], bj["ny"], bj["nz"], bj["spacing"], bj["origin"])
        tt = tets.reshape(-1, 4)
        x = sim.eng.get_target_values(b.targets[0]).reshape(-1, 3)
        sel = rng.choice(len(tt), ns // 8, replace=False)
        for t in tt[sel]:
            dr = rest[t[1:]] - rest[t[0]]          # rows: edges
            binv = np.linalg.inv(dr)               # (D_rest)^-1: fi = D binv
            vol = abs(np.linalg.det(dr)) / 6
            D = x[t[1:]] - x[t[0]]
            fi = D @ binv
            f = fi.reshape(-1)
            ic = f @ f
            J = np.linalg.det(fi)
            cf = np.array([[fi[1, 1] * fi[2, 2] - fi[1, 2] * fi[2, 1], fi[1, 2] * fi[2, 0] - fi[1, 0] * fi[2, 2],
                            fi[1, 0] * fi[2, 1] - fi[1, 1] * fi[2, 0]],
                           [fi[0, 2] * fi[2, 1] - fi[0, 1] * fi[2, 2], fi[0, 0] * fi[2, 2] - fi[0, 2] * fi[2, 0],
                            fi[0, 1] * fi[2, 0] - fi[0, 0] * fi[2, 1]],
                           [fi[0, 1] * fi[1, 2] - fi[0, 2] * fi[1, 1], fi[0, 2] * fi[1, 0] - fi[0, 0] * fi[1, 2],
                            fi[0, 0] * fi[1, 1] - fi[0, 1] * fi[1, 0]]]).reshape(-1)
            vw = vol * w
            ip1 = 1 / (ic + 1)
            c1, c2, c3, c4 = vw * mu * (1 - ip1), vw * 2 * mu * ip1 * ip1, vw * lam, vw * lam * (J - alpha)
            A = c1 * np.eye(9) + c2 * np.outer(f, f) + c3 * np.outer(cf, cf)
            for i in range(3):
                for ip in range(3):
                    if i == ip:
                        continue
                    for j in range(3):
                        for jp in range(3):
                            if j == jp:
                                continue
                            bb, d = 3 - i - ip, 3 - j - jp
                            s1 = 1 if (ip - i) % 3 == 1 else -1
                            s2 = 1 if (jp - j) % 3 == 1 else -1
                            A[3 * i + j, 3 * ip + jp] += c4 * s1 * s2 * fi[bb, d]
            K = np.kron(np.eye(3), binv.T)          # H_D = K^T A K  (index 3*edge + coord)
            out.append((K.T @ A @ K, D.copy()))
    return out


def proj_exact(M):
    l, V = np.linalg.eigh(M)
    return (V * np.maximum(l, 0)) @ V.T, l


def ldl(M):
    n = 9
    L = np.eye(n)
    d = np.zeros(n)
    for j in range(n):
        d[j] = M[j, j] - (L[j, :j] ** 2 * d[:j]).sum()
        for i in range(j + 1, n):
            L[i, j] = (M[i, j] - (L[i, :j] * L[j, :j] * d[:j]).sum()) / d[j]
    return L, d


W0 = np.linalg.qr(np.random.default_rng(1).standard_normal((9, 3)))[0]


def rot_start(D):
    W = np.zeros((9, 3))
    for a in range(3):
        e = np.zeros(3)
        e[a] = 1
        for i in range(3):
            W[3 * i:3 * i + 3, a] = np.cross(e, D[i])
    return np.linalg.qr(W)[0]


def proj_subspace(M, iters, D=None, tol_res=1e-11, delta=1e-11):
    nrm = np.linalg.norm(M)
    L, d = ldl(M)
    if np.any(np.abs(d) < 1e-300):
        return None, "pivot"
    W = W0.copy() if D is None else rot_start(D)
    for _ in range(iters):
        X = np.linalg.solve(L.T, np.linalg.solve(L, W) / d[:, None])
        W = np.linalg.qr(X)[0]
    S = W.T @ M @ W
    th, Vs = np.linalg.eigh(S)
    U = W @ Vs
    R = M @ U - U * th
    P = M.copy()
    for k in range(3):
        if th[k] < 0:
            if np.linalg.norm(R[:, k]) > tol_res * nrm:
                return None, "residual"
            P -= th[k] * np.outer(U[:, k], U[:, k])
    try:
        np.linalg.cholesky(P + delta * nrm * np.eye(9))
    except np.linalg.LinAlgError:
        return None, "psd"
    return P, "ok"


HD = sample_hd() if __name__ == "__main__" or os.environ.get("EVD_SAMPLE") else []
if __name__ == "__main__":
    H = [m for m, _ in HD]
    print("samples", len(H))
    neg = []
    for M in H:
        l = np.linalg.eigvalsh(M)
        neg.append((l < 0).sum())
    neg = np.array(neg)
    print("negative eigenvalue counts:", {int(k): int((neg == k).sum()) for k in np.unique(neg)})
    ls = np.array([np.linalg.eigvalsh(M) for M in H])
    nr = np.linalg.norm(H, axis=(1, 2))
    print("lambda_3/||M|| median", np.median(np.abs(ls[:, 2]) / nr), "lambda_4/||M|| median", np.median(np.abs(ls[:, 3]) / nr))
    for start, iters in [("rand", 5), ("rand", 7), ("rot", 3), ("rot", 4), ("rot", 5), ("rot", 6)]:
        res = {}
        err = 0.0
        for M, D in HD:
            P, why = proj_subspace(M, iters, D if start == "rot" else None)
            res[why] = res.get(why, 0) + 1
            if P is not None:
                Pe, _ = proj_exact(M)
                err = max(err, np.abs(P - Pe).max() / np.abs(Pe).max())
        print(f"{start} iters {iters}: {res} max rel err {err:.2e}", flush=True)

    if os.environ.get("TRACE"):
        for M, D in HD[:6]:
            nrm = np.linalg.norm(M)
            l = np.linalg.eigvalsh(M)
            L, d = ldl(M)
            W = rot_start(D)
            line = []
            for it in range(10):
                X = np.linalg.solve(L.T, np.linalg.solve(L, W) / d[:, None])
                W = np.linalg.qr(X)[0]
                S = W.T @ M @ W
                th, Vs = np.linalg.eigh(S)
                U = W @ Vs
                R = M @ U - U * th
                line.append(np.linalg.norm(R, axis=0).max() / nrm)
            print("eig/|M|", np.round(l[:5] / nrm, 6), "res:", " ".join(f"{v:.0e}" for v in line))
