"""Telescoping HBS factorization held in packed per-level device buffers.

Drop-in for the reference's `HbsFactorization` (factorization.py:25-86): the
same attributes (`tree`, `rank`, `u_bases`, `v_bases`, `discs`, `root_disc`,
`n`, `validate()`), but the blocks live on the GPU in the layout the kernels
produce (include/hbs_b200.h):

  level l:  U_l, V_l : (rows_l x r)   box j at rows [row_begin_l[j], row_begin_l[j+1])
            D_l      : flat, box j's rows_j x rows_j block at sq_off_l[j]
  root   :  (2r x 2r)

`u_bases[node_id]` etc. are read-only mappings that copy one whole level to
the host on first access (numpy float64, like the reference's dict values).
`apply_matrix` is the HBS sampler (factorization.py:89-143) on the device.
"""

from collections.abc import Mapping

import numpy as np
import torch

from . import _native
from .errors import DimensionError
from .tree import ClusterTree

_ORTHONORMALITY_TOL = 1e-10   # factorization.py:22


class LevelGeometry:
    """Device-side row geometry of one tree level (int64 tensors)."""

    def __init__(self, begins: np.ndarray, device):
        begins = np.asarray(begins, dtype=np.int64)
        sizes = np.diff(begins)
        self.nbox = sizes.size
        self.max_rows = int(sizes.max())
        self.min_rows = int(sizes.min())
        self.total_rows = int(begins[-1] - begins[0])
        sq = np.zeros(self.nbox + 1, dtype=np.int64)
        np.cumsum(sizes * sizes, out=sq[1:])
        self.sq_total = int(sq[-1])
        self.begins_host = begins
        self.sq_host = sq
        self.row_begin = torch.from_numpy(begins - begins[0]).to(device)
        self.sq_off = torch.from_numpy(sq).to(device)

    @classmethod
    def slice_of(cls, parent: "LevelGeometry", first: int, nbox: int) -> "LevelGeometry":
        """Geometry of boxes [first, first + nbox) of `parent`, with the device
        arrays derived from the parent's on the device (two tiny kernels on
        the current stream, no host-to-device copy: the host pipeline builds
        one of these per subtree and level while gigabytes of samples are in
        flight on the copy engine)."""
        g = cls.__new__(cls)
        begins = parent.begins_host[first:first + nbox + 1]
        sizes = np.diff(begins)
        g.nbox = nbox
        g.max_rows, g.min_rows = int(sizes.max()), int(sizes.min())
        g.total_rows = int(begins[-1] - begins[0])
        g.begins_host = begins
        g.sq_host = parent.sq_host[first:first + nbox + 1] - parent.sq_host[first]
        g.sq_total = int(g.sq_host[-1])
        g.row_begin = parent.row_begin[first:first + nbox + 1] - parent.row_begin[first:first + 1]
        g.sq_off = parent.sq_off[first:first + nbox + 1] - parent.sq_off[first:first + 1]
        return g


def tree_geometry(tree: ClusterTree, rank: int, device):
    """Geometry of levels 0..L: the leaf level uses the tree's ranges, coarser
    levels the packed 2r-row lifted blocks (compress.py:222-227)."""
    geo = [None] * (tree.depth + 1)
    geo[tree.depth] = LevelGeometry(tree.level_begin(tree.depth), device)
    for level in range(tree.depth - 1, -1, -1):
        geo[level] = LevelGeometry(np.arange((1 << level) + 1, dtype=np.int64) * 2 * rank, device)
    return geo


class _LevelBlocks(Mapping):
    """node id -> numpy block, materialising a whole level per first touch."""

    def __init__(self, fact, kind):
        self._f, self._kind = fact, kind

    def __getitem__(self, node_id):
        f = self._f
        level = int(node_id + 1).bit_length() - 1
        if node_id < 1 or level > f.tree.depth:
            raise KeyError(node_id)
        j = node_id - ((1 << level) - 1)
        host = f._host_level(level, self._kind)
        g = f.geometry[level]
        lo, hi = int(g.begins_host[j] - g.begins_host[0]), int(g.begins_host[j + 1] - g.begins_host[0])
        if self._kind == "d":
            rows = hi - lo
            return host[g.sq_host[j]:g.sq_host[j + 1]].reshape(rows, rows)
        return host[lo:hi]

    def __iter__(self):
        return iter(range(1, (1 << (self._f.tree.depth + 1)) - 1))

    def __len__(self):
        return (1 << (self._f.tree.depth + 1)) - 2


class HbsFactorization:
    """Telescoping factorization of a square operator over a cluster tree."""

    def __init__(self, tree: ClusterTree, rank: int, u_bases, v_bases, discs, root_disc, device=None):
        """Reference-compatible constructor from per-node host blocks
        (factorization.py:33-40); packs them into the device layout."""
        self.tree, self.rank = tree, rank
        root = np.asarray(root_disc, dtype=np.float64)
        _check_shapes(tree, rank, u_bases, v_bases, discs, root)
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.geometry = tree_geometry(tree, rank, dev)
        self.levels = []
        for level in range(tree.depth + 1):
            if level == 0:
                self.levels.append(None)
                continue
            nodes = tree.nodes_at_level(level)
            u = np.concatenate([np.asarray(u_bases[nd.id], dtype=np.float64) for nd in nodes])
            v = np.concatenate([np.asarray(v_bases[nd.id], dtype=np.float64) for nd in nodes])
            d = np.concatenate([np.asarray(discs[nd.id], dtype=np.float64).ravel() for nd in nodes])
            self.levels.append(tuple(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (u, v, d)))
        self.root_device = torch.from_numpy(root.copy()).to(dev)
        self._host = {}

    @classmethod
    def from_device(cls, tree, rank, geometry, levels, root):
        """Wrap buffers produced by the device compressor (no copies)."""
        self = cls.__new__(cls)
        self.tree, self.rank = tree, rank
        self.geometry, self.levels, self.root_device = geometry, levels, root
        self._host = {}
        return self

    # -- reference attributes ------------------------------------------------
    @property
    def n(self) -> int:
        return self.tree.n

    @property
    def device(self):
        return self.root_device.device

    @property
    def root_disc(self) -> np.ndarray:
        if "root" not in self._host:
            self._host["root"] = self.root_device.cpu().numpy()
        return self._host["root"]

    @property
    def u_bases(self):
        return _LevelBlocks(self, "u")

    @property
    def v_bases(self):
        return _LevelBlocks(self, "v")

    @property
    def discs(self):
        return _LevelBlocks(self, "d")

    def _host_level(self, level, kind):
        key = (level, kind)
        if key not in self._host:
            t = self.levels[level]["uvd".index(kind)]
            self._host[key] = t.cpu().numpy()
        return self._host[key]

    def materialize(self) -> int:
        """Copy every block to pinned host memory (one stream, one sync) so the
        reference-style dict views are free afterwards.  Returns bytes copied."""
        pending, nbytes = [], 0
        for level in range(1, self.tree.depth + 1):
            for kind, t in zip("uvd", self.levels[level]):
                nbytes_t = t.numel() * 8
                if (level, kind) in self._host:      # already on the host (pipelined compress)
                    nbytes += nbytes_t
                    continue
                h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                h.copy_(t, non_blocking=True)
                pending.append(((level, kind), h))
                nbytes += nbytes_t
        root = torch.empty(self.root_device.shape, dtype=torch.float64, pin_memory=True)
        root.copy_(self.root_device, non_blocking=True)
        nbytes += root.numel() * 8
        torch.cuda.synchronize(self.device)
        for key, h in pending:
            self._host[key] = h.numpy()
        self._host["root"] = root.numpy()
        return nbytes

    def validate(self):
        """Orthonormality of every basis and finiteness of all blocks
        (factorization.py:69-86), evaluated on the device per level; the first
        failure is reported in the reference's order (level order; per node:
        column basis, row basis, discrepancy)."""
        r = self.rank
        eye = torch.eye(r, dtype=torch.float64, device=self.device)
        for level in range(1, self.tree.depth + 1):
            g = self.geometry[level]
            u, v, d = self.levels[level]
            sizes = np.diff(g.begins_host)
            defects = []
            for basis in (u, v):
                if (sizes == sizes[0]).all():
                    blocks = basis.view(g.nbox, int(sizes[0]), r)
                    defects.append(torch.linalg.matrix_norm(blocks.transpose(1, 2) @ blocks - eye))
                else:
                    b0 = g.begins_host[0]
                    defects.append(torch.stack([torch.linalg.matrix_norm(basis[a - b0:b - b0].T @ basis[a - b0:b - b0] - eye)
                                                for a, b in zip(g.begins_host[:-1], g.begins_host[1:])]))
            bad_u, bad_v = (~(x <= _ORTHONORMALITY_TOL) for x in defects)
            bad_d = torch.zeros(g.nbox, dtype=torch.bool, device=self.device)
            nonfinite = torch.nonzero(~torch.isfinite(d)).reshape(-1)
            if nonfinite.numel():
                sq = torch.as_tensor(g.sq_host, device=self.device)
                bad_d[torch.searchsorted(sq, nonfinite, right=True) - 1] = True
            any_bad = bad_u | bad_v | bad_d
            if bool(any_bad.any()):
                j = int(torch.nonzero(any_bad)[0, 0])
                nid = (1 << level) - 1 + j
                if bool(bad_u[j]):
                    raise ValueError(f"node {nid}: column basis orthonormality defect {float(defects[0][j]):.3e}")
                if bool(bad_v[j]):
                    raise ValueError(f"node {nid}: row basis orthonormality defect {float(defects[1][j]):.3e}")
                raise ValueError(f"node {nid}: discrepancy block has non-finite entries")
        if not bool(torch.isfinite(self.root_device).all()):
            raise ValueError("root core has non-finite entries")
        return self

    def storage_floats(self) -> int:
        """Total stored floats (the `storage` count of factorization.py:193-203)."""
        total = self.root_device.numel()
        for level in range(1, self.tree.depth + 1):
            total += sum(t.numel() for t in self.levels[level])
        return total


def _check_shapes(tree, r, u_bases, v_bases, discs, root):
    """Block shapes of factorization.py:49-67."""
    if root.shape != (2 * r, 2 * r):
        raise DimensionError(f"root core must be {2 * r} x {2 * r}, got {root.shape}")
    for node in tree.nodes[1:]:
        rows = node.size if node.is_leaf else 2 * r
        for blocks, shape, kind in ((u_bases, (rows, r), "column basis"), (v_bases, (rows, r), "row basis"),
                                    (discs, (rows, rows), "discrepancy")):
            got = np.shape(blocks[node.id])
            if tuple(got) != shape:
                raise DimensionError(f"node {node.id}: {kind} must be {shape[0]} x {shape[1]}, got {tuple(got)}")


def _as_device(q, device):
    if isinstance(q, torch.Tensor):
        return q.to(device=device, dtype=torch.float64).contiguous(), False
    return torch.from_numpy(np.ascontiguousarray(q, dtype=np.float64)).to(device), True


def apply_matrix(f: HbsFactorization, q, transpose: bool = False, out=None, stream=None):
    """A q (or A^T q) for the columns of q through the telescoping factorization
    (factorization.py:89-143), on the device.  numpy in -> numpy out; torch in
    -> torch out (same device as the factorization)."""
    if q.ndim != 2 or q.shape[0] != f.n:
        raise DimensionError(f"expected a {f.n} x c matrix, got array of shape {tuple(q.shape)}")
    qd, to_host = _as_device(q, f.device)
    c = qd.shape[1]
    L, r = f.tree.depth, f.rank
    res = torch.empty_like(qd) if out is None else out
    ws_bytes = _workspace_bytes(L, r, c)
    ws = torch.empty(ws_bytes // 8 + 1, dtype=torch.float64, device=f.device)
    geo = f.geometry
    zero = 0
    rb = _native.ptr_array([zero] + [geo[l].row_begin.data_ptr() for l in range(1, L + 1)])
    sq = _native.ptr_array([zero] + [geo[l].sq_off.data_ptr() for l in range(1, L + 1)])
    us = _native.ptr_array([zero] + [f.levels[l][0].data_ptr() for l in range(1, L + 1)])
    vs = _native.ptr_array([zero] + [f.levels[l][1].data_ptr() for l in range(1, L + 1)])
    ds = _native.ptr_array([zero] + [f.levels[l][2].data_ptr() for l in range(1, L + 1)])
    st = stream if stream is not None else torch.cuda.current_stream(f.device).cuda_stream
    rc = _native.lib().hbs_apply(L, r, f.n, c, rb, sq, us, vs, ds, f.root_device.data_ptr(), qd.data_ptr(),
                                 res.data_ptr(), 1 if transpose else 0, ws.data_ptr(), ws_bytes, st)
    _native.check(rc, "hbs_apply")
    return res.cpu().numpy() if to_host else res


def _workspace_bytes(depth, r, c):
    import ctypes
    out = ctypes.c_size_t()
    _native.check(_native.lib().hbs_apply_workspace_bytes(depth, r, c, ctypes.byref(out)), "workspace")
    return out.value


def apply(f: HbsFactorization, q):
    """A q for one vector (factorization.py:146-151)."""
    q = np.asarray(q, dtype=np.float64)
    if q.ndim != 1 or q.shape[0] != f.n:
        raise DimensionError(f"expected a length-{f.n} vector, got array of shape {q.shape}")
    return apply_matrix(f, q[:, None])[:, 0]


def apply_transpose(f: HbsFactorization, q):
    """A^T q for one vector (factorization.py:154-159)."""
    q = np.asarray(q, dtype=np.float64)
    if q.ndim != 1 or q.shape[0] != f.n:
        raise DimensionError(f"expected a length-{f.n} vector, got array of shape {q.shape}")
    return apply_matrix(f, q[:, None], transpose=True)[:, 0]
