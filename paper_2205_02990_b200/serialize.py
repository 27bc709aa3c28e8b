"""`.hbsf` container I/O straight from / to the packed device layout.

Byte-compatible with the reference format (`pkg/src/hbs/serialize.py:1-91`):
header `<4sIQIII` (magic "HBSF", version 1, n, rank, depth, leaf threshold),
one little-endian u32 row count per non-root node in level order, then for
each non-root node in level order its U, V and D as column-major
little-endian float64, and the root core last.  Round trips are bit-exact
and files interchange with the reference in both directions.

Instead of walking per-node dicts, a whole level is re-laid out on its
device (one transpose + concatenation) and copied in one transfer.
"""

import struct

import numpy as np
import torch

from .errors import FormatError
from .factorization import HbsFactorization, tree_geometry
from .tree import build_tree

MAGIC = b"HBSF"
FORMAT_VERSION = 1
_HEADER = struct.Struct("<4sIQIII")


def _level_payload(u, v, d, sizes, r):
    """Bytes of one level: per box [U | V | D], each column-major f64."""
    if (sizes == sizes[0]).all():
        q = int(sizes[0])
        nb = sizes.size
        uu = u.reshape(nb, q, r).transpose(1, 2).reshape(nb, q * r)
        vv = v.reshape(nb, q, r).transpose(1, 2).reshape(nb, q * r)
        dd = d.reshape(nb, q, q).transpose(1, 2).reshape(nb, q * q)
        return torch.cat([uu, vv, dd], dim=1).contiguous().cpu().numpy().astype("<f8", copy=False).tobytes()
    parts, row, sq = [], 0, 0
    uh, vh, dh = (t.cpu().numpy() for t in (u, v, d))
    for q in sizes:
        q = int(q)
        parts += [uh[row:row + q].tobytes(order="F"), vh[row:row + q].tobytes(order="F"),
                  dh[sq:sq + q * q].reshape(q, q).tobytes(order="F")]
        row, sq = row + q, sq + q * q
    return b"".join(parts)


def save_factorization(f: HbsFactorization, path) -> None:
    """Write `f` in the reference's `.hbsf` layout."""
    tree, r = f.tree, f.rank
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(MAGIC, FORMAT_VERSION, tree.n, r, tree.depth, tree.leaf_threshold))
        rows = np.concatenate([f.geometry[lv].begins_host[1:] - f.geometry[lv].begins_host[:-1]
                               for lv in range(1, tree.depth + 1)]).astype("<u4")
        fh.write(rows.tobytes())
        for lv in range(1, tree.depth + 1):
            u, v, d = f.levels[lv]
            fh.write(_level_payload(u, v, d, np.diff(f.geometry[lv].begins_host), r))
        fh.write(np.asarray(f.root_disc, dtype="<f8").tobytes(order="F"))


def load_factorization(path, device=None) -> HbsFactorization:
    """Read a `.hbsf` file into the packed layout on `device` (default cuda);
    FormatError on bad magic, unknown version, inconsistent header or
    truncation (serialize.py:48-91)."""
    with open(path, "rb") as fh:
        buf = fh.read()
    if len(buf) < _HEADER.size:
        raise FormatError(f"truncated file: header needs {_HEADER.size} bytes past offset 0")
    magic, version, n, rank, depth, leaf_threshold = _HEADER.unpack_from(buf, 0)
    if magic != MAGIC:
        raise FormatError(f"bad magic {magic!r}, expected {MAGIC!r}")
    if version != FORMAT_VERSION:
        raise FormatError(f"unsupported format version {version}")
    tree = build_tree(n, leaf_threshold)
    if tree.depth != depth:
        raise FormatError(f"header depth {depth} does not match the depth-{tree.depth} tree for "
                          f"n={n}, leaf threshold {leaf_threshold}")
    off = _HEADER.size
    nnodes = (1 << (depth + 1)) - 2
    if off + 4 * nnodes > len(buf):
        raise FormatError(f"truncated file: node dimensions need {4 * nnodes} bytes past offset {off}")
    rows = np.frombuffer(buf, dtype="<u4", count=nnodes, offset=off)
    off += 4 * nnodes
    expected = np.concatenate([tree.level_sizes(lv) if lv == depth else np.full(1 << lv, 2 * rank)
                               for lv in range(1, depth + 1)])
    bad = np.nonzero(rows != expected)[0]
    if bad.size:
        i = int(bad[0])
        raise FormatError(f"node {i + 1}: header row count {rows[i]} does not match {expected[i]}")
    dev = torch.device(device) if device is not None else torch.device("cuda")
    levels = [None]
    r = rank
    for lv in range(1, depth + 1):
        sizes = tree.level_sizes(lv) if lv == depth else np.full(1 << lv, 2 * r)
        nbytes = int(8 * (2 * r * sizes.sum() + (sizes * sizes).sum()))
        if off + nbytes > len(buf):
            raise FormatError(f"truncated file: level {lv} blocks need {nbytes} bytes past offset {off}")
        raw = np.frombuffer(buf, dtype="<f8", count=nbytes // 8, offset=off)
        off += nbytes
        if (sizes == sizes[0]).all():
            q, nb = int(sizes[0]), sizes.size
            blk = torch.from_numpy(raw.copy()).to(dev).reshape(nb, 2 * q * r + q * q)
            u = blk[:, :q * r].reshape(nb, r, q).transpose(1, 2).reshape(nb * q, r).contiguous()
            v = blk[:, q * r:2 * q * r].reshape(nb, r, q).transpose(1, 2).reshape(nb * q, r).contiguous()
            d = blk[:, 2 * q * r:].reshape(nb, q, q).transpose(1, 2).reshape(-1).contiguous()
        else:
            us, vs, ds, pos = [], [], [], 0
            for q in sizes:
                q = int(q)
                us.append(raw[pos:pos + q * r].reshape(q, r, order="F")); pos += q * r
                vs.append(raw[pos:pos + q * r].reshape(q, r, order="F")); pos += q * r
                ds.append(raw[pos:pos + q * q].reshape(q, q, order="F").ravel()); pos += q * q
            u, v, d = (torch.from_numpy(np.ascontiguousarray(np.concatenate(x))).to(dev) for x in (us, vs, ds))
        levels.append((u, v, d))
    nroot = 8 * 4 * r * r
    if off + nroot > len(buf):
        raise FormatError(f"truncated file: root core needs {nroot} bytes past offset {off}")
    root = np.frombuffer(buf, dtype="<f8", count=4 * r * r, offset=off).reshape(2 * r, 2 * r, order="F")
    off += nroot
    if off != len(buf):
        raise FormatError(f"{len(buf) - off} trailing bytes after root core")
    return HbsFactorization.from_device(tree, r, tree_geometry(tree, r, dev), levels,
                                        torch.from_numpy(np.ascontiguousarray(root)).to(dev))
