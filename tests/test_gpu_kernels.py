"""GPU kernel-level parity through the C-ABI building blocks: the batched
Householder QR (reference: numpy.linalg.qr / LAPACK dgeqrf, as called by
nullspace(), linalg.py:52-62)."""
import ctypes

import numpy as np
import pytest
import torch

from paper_2205_02990_b200 import _native

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _native.lib()


def probe_qr(blocks, s):
    """Run hbs_probe_qr on a list of (rows x s) probe blocks (uneven sizes allowed)."""
    rows = [b.shape[0] for b in blocks]
    nr = max(rows)
    begins = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
    sq = np.concatenate([[0], np.cumsum(np.array(rows) ** 2)]).astype(np.int64)
    nbox = len(blocks)
    dev = torch.device("cuda")
    om = torch.from_numpy(np.concatenate(blocks)).to(dev)
    rb, so = torch.from_numpy(begins).to(dev), torch.from_numpy(sq).to(dev)
    npan = (nr + 31) // 32
    vt = torch.zeros(nbox, nr, s, dtype=torch.float64, device=dev)
    r = torch.zeros(nbox, nr, nr, dtype=torch.float64, device=dev)
    tau = torch.zeros(nbox, nr, dtype=torch.float64, device=dev)
    t = torch.zeros(nbox, npan, 32, 32, dtype=torch.float64, device=dev)
    rinv = torch.zeros(nbox, npan, 32, 32, dtype=torch.float64, device=dev)
    st = torch.zeros(nbox, dtype=torch.int32, device=dev)
    sz = ctypes.c_size_t()
    _native.check(_native.lib().hbs_probe_qr_scratch_bytes(nbox, nr, s, ctypes.byref(sz)), "scratch")
    scratch = torch.empty(max(sz.value // 8, 1), dtype=torch.float64, device=dev)
    rc = _native.lib().hbs_probe_qr(nbox, rb.data_ptr(), so.data_ptr(), nr, s, 1e-10, om.data_ptr(), vt.data_ptr(),
                                    r.data_ptr(), tau.data_ptr(), t.data_ptr(), rinv.data_ptr(),
                                    scratch.data_ptr() if sz.value else 0, st.data_ptr(),
                                    torch.cuda.current_stream().cuda_stream)
    _native.check(rc, "hbs_probe_qr")
    torch.cuda.synchronize()
    return [x.cpu().numpy() for x in (vt, r, tau, t, rinv, st)]


@pytest.mark.parametrize("rows,s", [(128, 192), (64, 96), (32, 48), (40, 120), (144, 216), (21, 45), (7, 30)])
def test_probe_qr_matches_lapack(rows, s):
    rng = np.random.default_rng(rows * 1000 + s)
    blocks = [rng.standard_normal((rows, s)) for _ in range(5)]
    vt, r, tau, t, rinv, st = probe_qr(blocks, s)
    assert not st.any()
    for b, om in enumerate(blocks):
        n = om.shape[0]
        # LAPACK (numpy) complete QR of omega^T: same reflectors => same R and Q
        q_ref, r_ref = np.linalg.qr(om.T, mode="complete")
        R = r[b][:n, :n]
        assert np.abs(R - r_ref[:n, :n]).max() <= 1e-12 * np.abs(r_ref).max()
        q = np.eye(s)
        for j in range(n - 1, -1, -1):
            v = vt[b][j]
            q -= tau[b][j] * np.outer(v, v @ q)
        assert np.abs(q - q_ref).max() <= 1e-12
        assert np.linalg.norm(q.T @ q - np.eye(s)) <= 1e-13 * s
        # the trailing ("last r columns") null basis equals the reference's nullspace()
        assert np.abs(om @ q[:, n:]).max() <= 1e-12 * np.abs(om).max()
        # compact-WY T blocks and diagonal-block inverses
        for p in range((n + 31) // 32):
            j0, nbp = 32 * p, min(32, n - 32 * p)
            V = vt[b][j0:j0 + nbp].T
            Hblk = np.eye(s) - V @ t[b][p][:nbp, :nbp] @ V.T
            Hseq = np.eye(s)
            for j in range(j0, j0 + nbp):
                Hseq = Hseq @ (np.eye(s) - tau[b][j] * np.outer(vt[b][j], vt[b][j]))
            assert np.abs(Hblk - Hseq).max() <= 1e-13
            Rb = R[j0:j0 + nbp, j0:j0 + nbp]
            assert np.abs(rinv[b][p][:nbp, :nbp] @ Rb - np.eye(nbp)).max() <= 1e-12


def test_probe_qr_flags_rank_deficiency():
    rng = np.random.default_rng(5)
    om = rng.standard_normal((16, 40))
    om[3] = om[0]
    ok = rng.standard_normal((16, 40))
    *_, st = probe_qr([ok, om, ok], 40)
    assert list(st) == [0, 1, 0]


def test_probe_qr_zero_block():
    vt, r, tau, t, rinv, st = probe_qr([np.zeros((8, 20))], 20)
    assert st[0] == 1          # sigma_max == 0 -> rank deficient (linalg.py:73)
    assert not np.any(tau)     # dlarfg: zero column -> tau = 0, H = I


def basis_qr(blocks, r):
    rows = [b.shape[0] for b in blocks]
    nr = max(rows)
    begins = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
    sq = np.concatenate([[0], np.cumsum(np.array(rows) ** 2)]).astype(np.int64)
    dev = torch.device("cuda")
    bb = torch.from_numpy(np.concatenate(blocks)).to(dev)
    q = torch.zeros_like(bb)
    rb, so = torch.from_numpy(begins).to(dev), torch.from_numpy(sq).to(dev)
    sz = ctypes.c_size_t()
    _native.check(_native.lib().hbs_basis_qr_scratch_bytes(len(blocks), nr, r, ctypes.byref(sz)), "scratch")
    scratch = torch.empty(max(sz.value // 8, 1), dtype=torch.float64, device=dev)
    rc = _native.lib().hbs_basis_qr(len(blocks), rb.data_ptr(), so.data_ptr(), nr, r, bb.data_ptr(), q.data_ptr(),
                                    scratch.data_ptr() if sz.value else 0, torch.cuda.current_stream().cuda_stream)
    _native.check(rc, "hbs_basis_qr")
    torch.cuda.synchronize()
    out, qh = [], q.cpu().numpy()
    for j in range(len(blocks)):
        out.append(qh[begins[j]:begins[j + 1]])
    return out


@pytest.mark.parametrize("rows,r", [(32, 16), (21, 8), (128, 64), (64, 32), (48, 24), (144, 72), (30, 15), (40, 40)])
def test_basis_qr_matches_lapack(rows, r):
    """col() building block: reduced QR with explicit Q (linalg.py:35-49)."""
    rng = np.random.default_rng(rows * 100 + r)
    blocks = [rng.standard_normal((rows, r)) for _ in range(3)]
    blocks.append(np.zeros((rows, r)))                      # zero block: Q = leading identity columns
    low = rng.standard_normal((rows, 2)) @ rng.standard_normal((2, r))
    blocks.append(low)                                      # rank-deficient block (oversampled case)
    qs = basis_qr(blocks, r)
    for b, q in zip(blocks, qs):
        q_ref = np.linalg.qr(b)[0][:, :r]
        assert np.linalg.norm(q.T @ q - np.eye(r)) <= 1e-12 * r
        if np.linalg.matrix_rank(b) == r:
            assert np.abs(q - q_ref).max() <= 1e-11      # same reflectors => same Q (LAPACK signs)
        assert np.linalg.norm(b - q @ (q.T @ b)) <= 1e-12 * max(1.0, np.linalg.norm(b))


def basis_orth(blocks, r):
    rows = [b.shape[0] for b in blocks]
    nr = max(rows)
    begins = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
    sq = np.concatenate([[0], np.cumsum(np.array(rows) ** 2)]).astype(np.int64)
    dev = torch.device("cuda")
    bb = torch.from_numpy(np.concatenate(blocks)).to(dev)
    q = torch.zeros_like(bb)
    rb, so = torch.from_numpy(begins).to(dev), torch.from_numpy(sq).to(dev)
    flags = torch.zeros(len(blocks), dtype=torch.int32, device=dev)
    sz = ctypes.c_size_t()
    _native.check(_native.lib().hbs_basis_qr_scratch_bytes(len(blocks), nr, r, ctypes.byref(sz)), "scratch")
    scratch = torch.empty(max(sz.value // 8, 1), dtype=torch.float64, device=dev)
    rc = _native.lib().hbs_basis_orth(len(blocks), rb.data_ptr(), so.data_ptr(), nr, r, bb.data_ptr(), q.data_ptr(),
                                      flags.data_ptr(), scratch.data_ptr() if sz.value else 0,
                                      torch.cuda.current_stream().cuda_stream)
    _native.check(rc, "hbs_basis_orth")
    torch.cuda.synchronize()
    qh = q.cpu().numpy()
    return [qh[begins[j]:begins[j + 1]] for j in range(len(blocks))], flags.cpu().numpy()


@pytest.mark.parametrize("rows,r", [(128, 64), (32, 16), (64, 32), (80, 40), (21, 8), (120, 40), (40, 40), (96, 48)])
def test_basis_orth_cholqr2(rows, r):
    """CholeskyQR2 bases (cholqr.cu): orthonormal, same span as the reference's
    col() (linalg.py:35-49), hence the same projector as LAPACK's Q; the
    Householder kernel takes over for rank-deficient / very ill-conditioned blocks."""
    rng = np.random.default_rng(rows * 1000 + r)
    blocks = [rng.standard_normal((rows, r)) for _ in range(3)]
    u, _, vt = np.linalg.svd(rng.standard_normal((rows, r)), full_matrices=False)
    blocks.append((u * np.logspace(0, -5, r)) @ vt)          # kappa 1e5: second full Cholesky pass
    blocks.append(np.zeros((rows, r)))                       # breakdown -> Householder
    blocks.append(rng.standard_normal((rows, 2)) @ rng.standard_normal((2, r)))   # rank 2 -> Householder
    blocks.append((u * np.logspace(0, -9, r)) @ vt)          # kappa 1e9 -> Householder
    qs, flags = basis_orth(blocks, r)
    assert list(flags[:4]) == [0, 0, 0, 0] and list(flags[4:]) == [1, 1, 1]
    for j, (b, q) in enumerate(zip(blocks, qs)):
        assert np.linalg.norm(q.T @ q - np.eye(r)) <= 1e-13 * r, j
        assert np.linalg.norm(b - q @ (q.T @ b)) <= 1e-13 * max(1.0, np.linalg.norm(b)), j
        if j < 4:
            q_ref = np.linalg.qr(b)[0]
            assert np.linalg.norm(q @ q.T - q_ref @ q_ref.T) <= 1e-12 * (1e5 if j == 3 else 1.0), j


def test_basis_orth_uneven_rows():
    rng = np.random.default_rng(11)
    blocks = [rng.standard_normal((n, 24)) for n in (24, 57, 128, 96, 31)]
    qs, flags = basis_orth(blocks, 24)
    assert not flags.any()
    for b, q in zip(blocks, qs):
        assert np.linalg.norm(q.T @ q - np.eye(24)) <= 1e-13 * 24
        assert np.linalg.norm(b - q @ (q.T @ b)) <= 1e-13 * np.linalg.norm(b)


def gram_factor(blocks, s, r):
    """hbs_gram_probe_factor on equal-size (rows x s) probe blocks."""
    rows = blocks[0].shape[0]
    nbox = len(blocks)
    dev = torch.device("cuda")
    om = torch.from_numpy(np.concatenate(blocks)).to(dev)
    rb = torch.arange(nbox + 1, dtype=torch.int64, device=dev) * rows
    npan = (rows + 31) // 32
    fac = torch.zeros(nbox, rows, s, dtype=torch.float64, device=dev)
    t = torch.zeros(nbox, npan, 32, 32, dtype=torch.float64, device=dev)
    flag = torch.full((nbox,), -1, dtype=torch.int32, device=dev)
    st = torch.full((nbox,), -1, dtype=torch.int32, device=dev)
    _native.check(_native.lib().hbs_gram_probe_factor(nbox, rb.data_ptr(), rows, s, r, om.data_ptr(), fac.data_ptr(),
                                                      t.data_ptr(), flag.data_ptr(), st.data_ptr(),
                                                      torch.cuda.current_stream().cuda_stream), "gram")
    torch.cuda.synchronize()
    return fac.cpu().numpy(), t.cpu().numpy(), flag.cpu().numpy(), st.cpu().numpy()


@pytest.mark.parametrize("rows,s", [(128, 192), (64, 96), (32, 48), (80, 120), (16, 40)])
def test_gram_factor_reproduces_householder(rows, s):
    """The Gram / Householder-reconstruction factorisation (gram_tm.cu) yields
    the LAPACK Householder reflectors, R and tau of Omega^T up to rounding
    (Householder QR is unique for dlarfg's sign rule)."""
    rng = np.random.default_rng(rows + s)
    r = s - rows
    blocks = [rng.standard_normal((rows, s)) for _ in range(3)]
    fac, t, flag, st = gram_factor(blocks, s, r)
    assert not flag.any() and not st.any()
    vt, rr, tau, tt, _, _ = probe_qr(blocks, s)
    for b in range(3):
        R = np.triu(fac[b][:, :rows].T)            # fac row j = column j of [R + V1; V2]
        assert np.abs(R - rr[b]).max() <= 1e-11 * np.abs(rr[b]).max()
        V = np.tril(fac[b].T, -1)[:, :rows] + np.eye(s, rows)
        Vref = vt[b].T
        assert np.abs(V - Vref).max() <= 1e-10
        # tau (the diagonal of each panel's T) in row 0 of the panel's T block;
        # the fused kernel forms T itself from V and tau
        for p in range((rows + 31) // 32):
            nbp = min(32, rows - 32 * p)
            assert np.abs(t[b][p][0][:nbp] - tau[b][32 * p:32 * p + nbp]).max() <= 1e-11
