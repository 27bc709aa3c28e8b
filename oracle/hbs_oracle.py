"""CPU ORACLE (test infrastructure only -- see oracle/__init__.py).

A numpy restatement of the reference's black-box HBS compression hot path
(arXiv 2205.02990, Alg. 2) as implemented in `/root/reference/pkg/src/hbs`.
It makes the same LAPACK calls as the reference (numpy.linalg.qr complete /
reduced, numpy.linalg.svd) so it reproduces the reference's numerics, but it
is organised level-batched over packed per-level arrays -- the same geometry
the device kernels use -- instead of dicts of per-node dataclasses.

Pinning: `tests/test_oracle.py` checks this restatement against the real
reference (imported from /root/reference when present) and against the
committed golden fixtures in `tests/golden/` produced by
`oracle/make_golden.py` from the unmodified reference.
"""

import numpy as np

TOL_DEFAULT = 1e-10          # linalg.py:20
STREAM_OMEGA, STREAM_PSI, STREAM_POWER, STREAM_SYNTHETIC = 0, 1, 2, 3   # linalg.py:15-18


class ProbeRankError(Exception):
    """Raised with (level, box index) when a probe block fails the sigma test."""

    def __init__(self, level, box, ratio):
        super().__init__(f"level {level} box {box}: sigma_min/sigma_max = {ratio:.3e}")
        self.level, self.box, self.ratio = level, box, ratio


def gaussian(n, s, seed, stream=0):
    """Seeded N(0,1) n x s draw: PCG64 on SeedSequence(seed, spawn_key=(stream,))
    (linalg.py:23-32)."""
    gen = np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy=seed, spawn_key=(stream,))))
    return gen.standard_normal((n, s))


def null_basis(w, r):
    """r trailing columns of the complete Householder Q of w^T (linalg.py:52-62)."""
    q_full = np.linalg.qr(w.T, mode="complete")[0]
    return q_full[:, q_full.shape[1] - r:]


def col_basis(b, r):
    """Leading r columns of the reduced unpivoted QR of b (linalg.py:35-49)."""
    return np.linalg.qr(b)[0][:, :r]


def right_solve(b, m, tol):
    """b @ pinv(m) through a thin SVD of m, with the sigma-ratio screen of
    linalg.py:65-90.  Returns (x, ratio); x is None when the screen fails."""
    u, sig, vt = np.linalg.svd(m, full_matrices=False)
    ratio = sig[-1] / max(sig[0], np.finfo(float).tiny)
    if sig[0] == 0.0 or sig[-1] < tol * sig[0]:
        return None, ratio
    return ((b @ vt.T) / sig) @ u.T, ratio


def node_step(om, ps, y, z, r, tol):
    """Bases + discrepancy of one box (compress.py:155-197).  Returns u, v, d
    or raises ProbeRankError(level=None, box=None)."""
    u = col_basis(y @ null_basis(om, r), r)
    v = col_basis(z @ null_basis(ps, r), r)
    xy, ry = right_solve(y, om, tol)
    if xy is None:
        raise ProbeRankError(None, None, ry)
    xz, rz = right_solve(z, ps, tol)
    if xz is None:
        raise ProbeRankError(None, None, rz)
    # same association order as compress.py:195-197, so results are bitwise equal
    inside_u = xy - u @ (u.T @ xy)
    outside_v = u @ (u.T @ (xz - v @ (v.T @ xz)).T)
    return u, v, inside_u + outside_v


def lift_rows(u, v, d, om, ps, y, z):
    """One child's r-row share of the parent quadruple (compress.py:209-219)."""
    return (v.T @ om, u.T @ ps, u.T @ (y - d @ om), v.T @ (z - d.T @ ps))


class OracleFactorization:
    """Packed telescoping factorization: for level l = 1..L, lists indexed by
    the box position j (node id 2^l - 1 + j); `root` is the 2r x 2r core."""

    def __init__(self, bounds, rank, U, V, D, root):
        self.bounds, self.rank = bounds, rank
        self.U, self.V, self.D, self.root = U, V, D, root

    @property
    def depth(self):
        return len(self.bounds) - 1

    @property
    def n(self):
        return int(self.bounds[0][-1])

    def node_blocks(self, node_id):
        level = int(np.floor(np.log2(node_id + 1)))
        j = node_id - ((1 << level) - 1)
        return self.U[level][j], self.V[level][j], self.D[level][j]


def tree_depth(n, leaf):
    """Smallest L >= 1 with ceil(n / 2^L) <= leaf (tree.py:80-82)."""
    depth = 1
    while (n + (1 << depth) - 1) >> depth > leaf:
        depth += 1
    return depth


def level_bounds(n, depth):
    """Box row starts per level with the reference split rule (tree.py:84-100)."""
    out = [np.array([0, n], dtype=np.int64)]
    for _ in range(depth):
        b = out[-1]
        mid = b[:-1] + (b[1:] - b[:-1] + 1) // 2
        nxt = np.empty(2 * (b.size - 1) + 1, dtype=np.int64)
        nxt[0:-1:2], nxt[1:-1:2], nxt[-1] = b[:-1], mid, n
        out.append(nxt)
    return out


def compress(omega, psi, y, z, bounds, r, tol=TOL_DEFAULT):
    """Level sweep of compress_from_samples (compress.py:236-280) over packed
    quadruples.  Raises ProbeRankError(level, box) for the first failing box in
    the reference order (deepest level first, ascending position)."""
    depth = len(bounds) - 1
    s = omega.shape[1]
    U, V, D = [None] * (depth + 1), [None] * (depth + 1), [None] * (depth + 1)
    quad = (omega, psi, y, z)          # leaf level: the global samples
    rows_of = bounds[depth]
    for level in range(depth, 0, -1):
        nbox = 1 << level
        Ul, Vl, Dl = [], [], []
        lifted = [np.empty((nbox * r, s)) for _ in range(4)]
        for j in range(nbox):
            lo, hi = (rows_of[j], rows_of[j + 1]) if level == depth else (2 * r * j, 2 * r * (j + 1))
            blk = [m[lo:hi] for m in quad]
            try:
                u, v, d = node_step(*blk, r, tol)
            except ProbeRankError as exc:
                raise ProbeRankError(level, j, exc.ratio) from None
            Ul.append(u), Vl.append(v), Dl.append(d)
            for dst, part in zip(lifted, lift_rows(u, v, d, *blk)):
                dst[j * r:(j + 1) * r] = part
        U[level], V[level], D[level] = Ul, Vl, Dl
        quad = tuple(lifted)
    root, ratio = right_solve(quad[2], quad[0], tol)          # compress.py:230-233
    if root is None:
        raise ProbeRankError(0, 0, ratio)
    return OracleFactorization(bounds, r, U, V, D, root)


def apply(f, q, transpose=False):
    """Telescoping apply, up / root / down sweeps (factorization.py:89-143)."""
    q = np.asarray(q, dtype=np.float64)
    vec = q.ndim == 1
    if vec:
        q = q[:, None]
    L, r = f.depth, f.rank
    up, down = (f.U, f.V) if transpose else (f.V, f.U)
    dmat = (lambda m: m.T) if transpose else (lambda m: m)
    rows = f.bounds[L]
    qhat = [None] * (L + 1)
    qhat[L] = np.concatenate([up[L][j].T @ q[rows[j]:rows[j + 1]] for j in range(1 << L)])
    for level in range(L - 1, 0, -1):
        qhat[level] = np.concatenate(
            [up[level][j].T @ qhat[level + 1][2 * r * j:2 * r * (j + 1)] for j in range(1 << level)])
    uhat = dmat(f.root) @ qhat[1]
    for level in range(1, L):
        uhat = np.concatenate(
            [down[level][j] @ uhat[r * j:r * (j + 1)] + dmat(f.D[level][j]) @ qhat[level + 1][2 * r * j:2 * r * (j + 1)]
             for j in range(1 << level)])
    out = np.concatenate(
        [down[L][j] @ uhat[r * j:r * (j + 1)] + dmat(f.D[L][j]) @ q[rows[j]:rows[j + 1]] for j in range(1 << L)])
    return out[:, 0] if vec else out


def dense(f):
    """Explicit matrix of a factorization (factorization.py:162-176); small n only."""
    import scipy.linalg
    core = f.root
    for level in range(1, f.depth + 1):
        ub = scipy.linalg.block_diag(*f.U[level])
        vb = scipy.linalg.block_diag(*f.V[level])
        db = scipy.linalg.block_diag(*f.D[level])
        core = ub @ core @ vb.T + db
    return core


# ---------------------------------------------------------------------------
# Synthetic inputs of BASELINE.json
# ---------------------------------------------------------------------------

def baseline_generator(n, leaf, k, seed=0, decay=None):
    """Exact-rank-k synthetic HBS operator on build_tree(n, leaf), as an
    OracleFactorization.  Per non-root node in level order: U, V = qr(N(0,1))
    (leaf rows or 2k rows); leaf D = N(0,1)/sqrt(m) + I; parent D =
    [[0, B1], [B2, 0]]; root [[0, B], [B', 0]]; B = N(0,1)/sqrt(k), or
    Q1 diag(decay^i) Q2^T when `decay` is given (config 4)."""
    depth = tree_depth(n, leaf)
    bounds = level_bounds(n, depth)
    gen = np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy=seed, spawn_key=(STREAM_SYNTHETIC,))))

    def coupling():
        if decay is None:
            return gen.standard_normal((k, k)) / np.sqrt(k)
        q1 = np.linalg.qr(gen.standard_normal((k, k)))[0]
        q2 = np.linalg.qr(gen.standard_normal((k, k)))[0]
        return (q1 * decay ** np.arange(k)) @ q2.T

    def off_diag(b1, b2):
        out = np.zeros((2 * k, 2 * k))
        out[:k, k:], out[k:, :k] = b1, b2
        return out

    U, V, D = [None] * (depth + 1), [None] * (depth + 1), [None] * (depth + 1)
    for level in range(1, depth + 1):
        sizes = np.diff(bounds[level]) if level == depth else np.full(1 << level, 2 * k)
        U[level], V[level], D[level] = [], [], []
        for rows in sizes:
            rows = int(rows)
            U[level].append(np.linalg.qr(gen.standard_normal((rows, k)))[0])
            V[level].append(np.linalg.qr(gen.standard_normal((rows, k)))[0])
            if level == depth:
                D[level].append(gen.standard_normal((rows, rows)) / np.sqrt(rows) + np.eye(rows))
            else:
                b1 = coupling()
                D[level].append(off_diag(b1, coupling()))
    b = coupling()
    root = off_diag(b, coupling())
    return OracleFactorization(bounds, k, U, V, D, root)


def ellipse_log_kernel(n):
    """Config 3 operator: x_i on the ellipse (cos t, 0.5 sin t), t = 2 pi i / n;
    A_ij = log|x_i - x_j| (i != j), A_ii = 1."""
    t = 2.0 * np.pi * np.arange(n) / n
    x = np.stack((np.cos(t), 0.5 * np.sin(t)), axis=1)
    diff = x[:, None, :] - x[None, :, :]
    dist = np.sqrt((diff ** 2).sum(-1))
    np.fill_diagonal(dist, 1.0)
    a = np.log(dist)
    np.fill_diagonal(a, 1.0)
    return a


def samples_from(f_or_dense, s, seed=0):
    """(omega, psi, y, z) = draw_samples(., s, seed) (compress.py:132-141)."""
    if isinstance(f_or_dense, np.ndarray):
        n = f_or_dense.shape[0]
        fwd = lambda x: f_or_dense @ x
        bwd = lambda x: f_or_dense.T @ x
    else:
        n = f_or_dense.n
        fwd = lambda x: apply(f_or_dense, x)
        bwd = lambda x: apply(f_or_dense, x, transpose=True)
    om = gaussian(n, s, seed, STREAM_OMEGA)
    ps = gaussian(n, s, seed, STREAM_PSI)
    return om, ps, fwd(om), bwd(ps)


def rel_apply_error(f_test, f_ref, x):
    """||(A_test - A_ref) x|| / ||A_ref x|| for apply-able operators or dense
    arrays (the parity metric of SURVEY.md section 8(c))."""
    def ap(f):
        return f @ x if isinstance(f, np.ndarray) else apply(f, x)
    ref = ap(f_ref)
    return float(np.linalg.norm(ap(f_test) - ref) / np.linalg.norm(ref))
