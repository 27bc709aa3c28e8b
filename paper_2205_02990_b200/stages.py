"""Per-node stages of the compressor as batch-of-one device calls -- the rest
of the reference's public API (pkg/src/hbs/__init__.py:53-90) around
compress_from_samples, so the reference's stage-by-stage usage
(test_compress.py:159-257) runs against the drop-in:

  NodeSamples, CompressedNode, leaf_node_samples, compress_node_bases,
  compute_discrepancy, lift_to_parent, compute_root   (compress.py:97-233)
  col, nullspace, lstsq_right                          (linalg.py:35-90)
  storage, StorageReport, LevelStorage                 (factorization.py:178-203)

Each call runs one box through the same kernels the level sweep uses
(hbs_probe_qr: LAPACK-convention Householder QR of Omega^T; hbs_basis_qr:
LAPACK-signed reduced QR), with the small products on the device.  Inputs may
be numpy arrays or CUDA tensors; outputs follow the inputs (numpy in ->
numpy out), as the reference returns numpy.  Shape checks, exception classes
and madd charges are the reference's.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .compress import DEFAULT_ILL_CONDITIONING_TOL, SampleSet
from .errors import ConfigurationError, DimensionError, IllConditionedProbeError
from .flops import add_madds, matmul_madds, qr_madds, svd_madds
from .tree import Node

_F64 = torch.float64


def _dev(x, device=None):
    if isinstance(x, torch.Tensor):
        return x.to(device=device or (x.device if x.is_cuda else "cuda"), dtype=_F64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(device or "cuda")


def _like(t, *refs):
    """numpy when every reference input was numpy, else the CUDA tensor."""
    if any(isinstance(r, torch.Tensor) for r in refs):
        return t
    return t.cpu().numpy()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _one_box(rows, device):
    rb = torch.tensor([0, rows], dtype=torch.int64, device=device)
    sq = torch.tensor([0, rows * rows], dtype=torch.int64, device=device)
    return rb, sq


def _probe_qr(m):
    """Householder QR of m^T (m: rows x cols, rows <= cols) on the device:
    reflectors (rows x cols, reflector j as row j), R, T blocks, status."""
    rows, cols = m.shape
    dev = m.device
    rb, sq = _one_box(rows, dev)
    npan = (rows + 31) // 32
    vt = torch.zeros(rows, cols, dtype=_F64, device=dev)
    r = torch.zeros(rows, rows, dtype=_F64, device=dev)
    tau = torch.zeros(rows, dtype=_F64, device=dev)
    t = torch.zeros(npan, 32, 32, dtype=_F64, device=dev)
    rinv = torch.zeros(npan, 32, 32, dtype=_F64, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = _native.lib()
    sz = ctypes.c_size_t()
    _native.check(lib.hbs_probe_qr_scratch_bytes(1, rows, cols, ctypes.byref(sz)), "probe scratch")
    scratch = torch.empty(max(sz.value // 8, 1), dtype=_F64, device=dev)
    _native.check(lib.hbs_probe_qr(1, rb.data_ptr(), sq.data_ptr(), rows, cols, 0.0, m.data_ptr(), vt.data_ptr(),
                                   r.data_ptr(), tau.data_ptr(), t.data_ptr(), rinv.data_ptr(),
                                   scratch.data_ptr() if sz.value else 0, st.data_ptr(), _stream()), "hbs_probe_qr")
    return vt, r, t


def _apply_q_left(vt, t, e):
    """Q e for Q = H_0 ... H_{n-1} (blocked: panel block reflectors, last first)."""
    rows = vt.shape[0]
    for p in range((rows + 31) // 32 - 1, -1, -1):
        j0, nbp = 32 * p, min(32, rows - 32 * p)
        v = vt[j0:j0 + nbp].T                        # cols x nbp, unit diagonal stored
        e = e - v @ (t[p, :nbp, :nbp] @ (v.T @ e))
    return e


def _apply_q_right(vt, t, b):
    """b Q (forward over the panels)."""
    rows = vt.shape[0]
    for p in range((rows + 31) // 32):
        j0, nbp = 32 * p, min(32, rows - 32 * p)
        v = vt[j0:j0 + nbp].T
        b = b - ((b @ v) @ t[p, :nbp, :nbp]) @ v.T
    return b


def nullspace(b, k: int):
    """k orthonormal columns of null(b) for a wide b: the trailing columns of
    the complete Householder Q of b^T (linalg.py:52-62)."""
    rows, cols = b.shape
    if cols - rows < k:
        raise DimensionError(f"a {rows} x {cols} matrix only guarantees nullity {max(cols - rows, 0)}, need {k}")
    add_madds(qr_madds(cols, rows, full=True))
    m = _dev(b)
    vt, _, t = _probe_qr(m)
    e = torch.zeros(cols, k, dtype=_F64, device=m.device)
    e[cols - k:] = torch.eye(k, dtype=_F64, device=m.device)
    return _like(_apply_q_left(vt, t, e), b)


def col(b, k: int):
    """k leading columns of the Q factor of the unpivoted reduced QR of b
    (linalg.py:35-49), LAPACK signs."""
    rows, cols = b.shape
    if k > min(rows, cols):
        raise DimensionError(f"cannot extract {k} basis columns from a {rows} x {cols} matrix")
    add_madds(qr_madds(rows, cols))
    bd = _dev(b)
    w = min(rows, cols)            # the Q of a wide b is that of its leading square block
    src = bd[:, :w].contiguous()
    dev = bd.device
    rb, sq = _one_box(rows, dev)
    q = torch.empty(rows, w, dtype=_F64, device=dev)
    lib = _native.lib()
    sz = ctypes.c_size_t()
    _native.check(lib.hbs_basis_qr_scratch_bytes(1, rows, w, ctypes.byref(sz)), "basis scratch")
    scratch = torch.empty(max(sz.value // 8, 1), dtype=_F64, device=dev)
    _native.check(lib.hbs_basis_qr(1, rb.data_ptr(), sq.data_ptr(), rows, w, src.data_ptr(), q.data_ptr(),
                                   scratch.data_ptr() if sz.value else 0, _stream()), "hbs_basis_qr")
    q = q[:, :k]
    if k == cols:
        scale = float(torch.linalg.norm(bd))
        assert scale == 0.0 or float(torch.linalg.norm(bd - q @ (q.T @ bd))) <= 1e-8 * scale
    return _like(q.contiguous(), b)


def lstsq_right(b, m, tol: float = DEFAULT_ILL_CONDITIONING_TOL):
    """X = B M^+ for a wide, full-row-rank M (linalg.py:65-90), through the
    Householder QR of M^T: X = (B Q)(:, :rows) R^{-T}.  The sigma test is
    the diag(R) screen of the level sweep (min|R_ii| < tol max|R_ii| raises;
    exact in the raising direction)."""
    m_rows, m_cols = m.shape
    if m_rows > m_cols:
        raise DimensionError(f"probe matrix must be wide, got {m_rows} x {m_cols}")
    if b.shape[1] != m_cols:
        raise DimensionError(f"column mismatch: B is {b.shape[0]} x {b.shape[1]}, M is {m_rows} x {m_cols}")
    add_madds(svd_madds(m_rows, m_cols))
    md, bd = _dev(m), _dev(b)
    vt, r, t = _probe_qr(md)
    diag = torch.abs(torch.diagonal(r))
    hi, lo = float(diag.max()), float(diag.min())
    if not hi > 0.0 or lo < tol * hi or not np.isfinite(hi):
        raise IllConditionedProbeError(
            f"probe matrix ({m_rows} x {m_cols}) is rank deficient within tolerance {tol:g} "
            f"(|R_ii| ratio = {lo / max(hi, np.finfo(float).tiny):.3e}); increase the probe count s")
    add_madds(matmul_madds(b.shape[0], m_cols, m_rows) + matmul_madds(b.shape[0], m_rows, m_rows))
    bq = _apply_q_right(vt, t, bd)[:, :m_rows]
    xt = torch.linalg.solve_triangular(r, bq.T.contiguous(), upper=True)   # R X^T = (B Q1)^T
    return _like(xt.T.contiguous(), b, m)


@dataclass(frozen=True)
class NodeSamples:
    """One node's rows of the probe quadruple (compress.py:97-118)."""
    omega_t: object
    psi_t: object
    y_t: object
    z_t: object

    def __post_init__(self):
        shapes = {tuple(self.omega_t.shape), tuple(self.psi_t.shape), tuple(self.y_t.shape), tuple(self.z_t.shape)}
        if len(shapes) != 1:
            raise DimensionError(f"node sample matrices must share one shape, got {shapes}")

    @property
    def rows(self) -> int:
        return self.omega_t.shape[0]

    @property
    def probes(self) -> int:
        return self.omega_t.shape[1]


@dataclass(frozen=True)
class CompressedNode:
    """Bases, discrepancy block and consumed samples of a node (compress.py:121-129)."""
    u: object
    v: object
    disc: object
    samples: NodeSamples


def leaf_node_samples(samples: SampleSet, node: Node) -> NodeSamples:
    """Row slices of the global quadruple for one leaf (compress.py:144-152)."""
    sl = slice(node.begin, node.end)
    return NodeSamples(omega_t=samples.omega[sl], psi_t=samples.psi[sl], y_t=samples.y[sl], z_t=samples.z[sl])


def compress_node_bases(ns: NodeSamples, r: int):
    """(u, v, p, q) of one node (compress.py:155-175)."""
    if ns.probes - ns.rows < r:
        raise ConfigurationError(
            f"probe count {ns.probes} leaves nullity {ns.probes - ns.rows} < rank {r} "
            f"for a {ns.rows}-row node; increase the probe count s")
    p = _dev(nullspace(_dev(ns.omega_t), r))
    add_madds(matmul_madds(ns.rows, ns.probes, r))
    u = col(_dev(ns.y_t) @ p, r)
    q = _dev(nullspace(_dev(ns.psi_t), r))
    add_madds(matmul_madds(ns.rows, ns.probes, r))
    v = col(_dev(ns.z_t) @ q, r)
    refs = (ns.omega_t,)
    return _like(u, *refs), _like(v, *refs), _like(p, *refs), _like(q, *refs)


def compute_discrepancy(u, v, ns: NodeSamples, tol: float = DEFAULT_ILL_CONDITIONING_TOL):
    """D = (I - UU^T) Y Omega^+ + UU^T ((I - VV^T) Z Psi^+)^T (compress.py:178-197)."""
    rows = ns.rows
    ys = _dev(lstsq_right(_dev(ns.y_t), _dev(ns.omega_t), tol))
    zs = _dev(lstsq_right(_dev(ns.z_t), _dev(ns.psi_t), tol))
    add_madds(6 * matmul_madds(u.shape[1], rows, rows))
    ud, vd = _dev(u), _dev(v)
    left = ys - ud @ (ud.T @ ys)
    right = ud @ (ud.T @ (zs - vd @ (vd.T @ zs)).T)
    return _like(left + right, u, ns.omega_t)


def lift_to_parent(alpha: CompressedNode, beta: CompressedNode) -> NodeSamples:
    """Parent test / sample rows from two compressed children (compress.py:200-227)."""
    def lifted(child):
        ns = child.samples
        rows, s = ns.rows, ns.probes
        r = child.u.shape[1]
        add_madds(4 * matmul_madds(r, rows, s) + 2 * matmul_madds(rows, rows, s))
        u, v, d = _dev(child.u), _dev(child.v), _dev(child.disc)
        om, ps, y, z = (_dev(m) for m in (ns.omega_t, ns.psi_t, ns.y_t, ns.z_t))
        return v.T @ om, u.T @ ps, u.T @ (y - d @ om), v.T @ (z - d.T @ ps)

    a, b = lifted(alpha), lifted(beta)
    ref = alpha.samples.omega_t
    return NodeSamples(*(_like(torch.cat((x, y)), ref) for x, y in zip(a, b)))


def compute_root(ns: NodeSamples, tol: float = DEFAULT_ILL_CONDITIONING_TOL):
    """Root core D_root = Y_root Omega_root^+ (compress.py:230-233)."""
    return lstsq_right(ns.y_t, ns.omega_t, tol)


@dataclass(frozen=True)
class LevelStorage:
    level: int
    basis_floats: int
    disc_floats: int


@dataclass(frozen=True)
class StorageReport:
    total_floats: int
    floats_per_dof: float
    levels: list


def storage(f) -> StorageReport:
    """Exact float counts per level and in total (factorization.py:193-203),
    from the packed device layout."""
    levels = [LevelStorage(level=0, basis_floats=0, disc_floats=int(f.root_device.numel()))]
    for level in range(1, f.tree.depth + 1):
        u, v, d = f.levels[level]
        levels.append(LevelStorage(level=level, basis_floats=int(u.numel() + v.numel()), disc_floats=int(d.numel())))
    total = sum(lv.basis_floats + lv.disc_floats for lv in levels)
    return StorageReport(total_floats=total, floats_per_dof=total / f.n, levels=levels)
