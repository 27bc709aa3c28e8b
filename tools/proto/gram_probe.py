"""Numerics prototype (dev tool) of the Gram / Cholesky + Householder-
reconstruction probe factorisation for nullity == r boxes, against the
LAPACK-path oracle.  Per box: G = Om Om^T = R^T R; LU of M1 = Om1^T - S R with
adaptive signs gives V1 (unit lower) and U'; V2 = Om2^T U'^-1;
T = -U' R^-1 S V1^-T; YH = Y - (Y V) T V^T; X = YH[:, :n] S R^-T; YP = YH[:, n:].
"""
import sys, os
import numpy as np
import scipy.linalg as sl
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from oracle import hbs_oracle as O


def gram_probe(om, y):
    n, s = om.shape
    G = om @ om.T
    R = np.linalg.cholesky(G).T          # upper
    M = om[:, :n].T.copy()                # n x n  (Om1^T)
    sg = np.zeros(n)
    L = np.eye(n)
    Up = np.zeros((n, n))
    A = M.copy()
    for i in range(n):
        a = A[i, i]
        sg[i] = -1.0 if a >= 0 else 1.0   # s_i = -sign(a)
        A[i, i:] -= sg[i] * R[i, i:]
        piv = A[i, i]
        L[i + 1:, i] = A[i + 1:, i] / piv
        A[i + 1:, i + 1:] -= np.outer(L[i + 1:, i], A[i, i + 1:])
        Up[i, i:] = A[i, i:]
    V2 = sl.solve_triangular(Up, om[:, n:], trans='T', lower=False).T  # Om2^T U'^-1 : (r x n)
    V = np.vstack([L, V2])
    # T = -U' R^-1 S V1^-T
    UR = sl.solve_triangular(R, Up.T, trans='T', lower=False).T        # U' R^-1
    T = -sl.solve_triangular(L, (UR * sg).T, lower=True, unit_diagonal=True).T
    H = np.eye(s) - V @ T @ V.T
    YH = y - ((y @ V) @ T) @ V.T
    X = (YH[:, :n] * sg) @ np.linalg.inv(R).T
    YP = YH[:, n:]
    return X, YP, H, R, sg


def check_node(n=128, s=192, seed=0):
    rng = np.random.default_rng(seed)
    om = rng.standard_normal((n, s)); y = rng.standard_normal((n, s))
    X, YP, H, R, sg = gram_probe(om, y)
    print("orth H", np.abs(H.T @ H - np.eye(s)).max(), " Om P", np.abs(om @ H[:, n:]).max(),
          " X err", np.abs(X - y @ np.linalg.pinv(om)).max() / np.abs(X).max(),
          " Q1 vs", np.abs(H[:, :n] * sg - om.T @ np.linalg.inv(R)).max())


def compress(omega, psi, y, z, bounds, r):
    depth = len(bounds) - 1
    s = omega.shape[1]
    U, V, D = [None] * (depth + 1), [None] * (depth + 1), [None] * (depth + 1)
    quad = (omega, psi, y, z)
    rows_of = bounds[depth]
    for level in range(depth, 0, -1):
        nbox = 1 << level
        Ul, Vl, Dl = [], [], []
        lifted = [np.empty((nbox * r, s)) for _ in range(4)]
        for j in range(nbox):
            lo, hi = (rows_of[j], rows_of[j + 1]) if level == depth else (2 * r * j, 2 * r * (j + 1))
            om, ps, yy, zz = [m[lo:hi] for m in quad]
            n = hi - lo
            if s - n == r:
                xy, yp, *_ = gram_probe(om, yy)
                xz, zq, *_ = gram_probe(ps, zz)
                u = np.linalg.qr(yp)[0]; v = np.linalg.qr(zq)[0]
            else:
                u = O.col_basis(yy @ O.null_basis(om, r), r)
                v = O.col_basis(zz @ O.null_basis(ps, r), r)
                xy = O.right_solve(yy, om, 1e-10)[0]; xz = O.right_solve(zz, ps, 1e-10)[0]
            d = xy - u @ (u.T @ xy) + u @ (u.T @ (xz - v @ (v.T @ xz)).T)
            Ul.append(u); Vl.append(v); Dl.append(d)
            for dst, part in zip(lifted, O.lift_rows(u, v, d, om, ps, yy, zz)):
                dst[j * r:(j + 1) * r] = part
        U[level], V[level], D[level] = Ul, Vl, Dl
        quad = tuple(lifted)
    root = O.right_solve(quad[2], quad[0], 1e-10)[0]
    return O.OracleFactorization(bounds, r, U, V, D, root)


if __name__ == "__main__":
    for sd in range(3):
        check_node(seed=sd)
    check_node(64, 96)
    for (n, leaf, k, r, s, decay) in [(2048, 128, 64, 72, 216, 0.9), (2048, 128, 64, 64, 192, 0.9),
                                      (4096, 64, 32, 40, 120, None), (4096, 64, 32, 32, 96, None),
                                      (16384, 128, 64, 64, 192, 0.9), (16384, 128, 64, 72, 216, 0.9)]:
        truth = O.baseline_generator(n, leaf, k, seed=0, decay=decay)
        om, ps, y, z = O.samples_from(truth, s, 0)
        depth = O.tree_depth(n, leaf)
        b = O.level_bounds(n, depth)
        x = O.gaussian(n, 4, 0, 4)
        tx = O.apply(truth, x)
        fg = compress(om, ps, y, z, b, r)
        fr = O.compress(om, ps, y, z, b, r)
        eg = np.linalg.norm(O.apply(fg, x) - tx) / np.linalg.norm(tx)
        er = np.linalg.norm(O.apply(fr, x) - tx) / np.linalg.norm(tx)
        print(f"n={n} r={r} s={s}: gram err {eg:.3e}  lapack err {er:.3e}")
