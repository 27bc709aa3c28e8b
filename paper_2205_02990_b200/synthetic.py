"""Device-side generators of the BASELINE.json synthetic operators
 for full-size runs (N = 2^20, 2^22) where the host
generator would take minutes.  Same construction as the oracle's
`baseline_generator` (exact block rank k; leaf D = N(0,1)/sqrt(m) + I;
parent D = [[0, B1], [B2, 0]]; optional singular-value decay of B) but drawn
from torch's CUDA Philox stream, so values differ from the host generator --
seeded synthetic inputs of the same shapes and distributions.  Test/bench
input generation only; not part of the compress path.
"""

import math

import numpy as np
import torch

from .factorization import HbsFactorization, tree_geometry
from .tree import ClusterTree


def _orthonormal(gen, batch, rows, k, device):
    a = torch.randn(batch, rows, k, generator=gen, dtype=torch.float64, device=device)
    return torch.linalg.qr(a).Q


def _coupling(gen, batch, k, decay, device):
    if decay is None:
        return torch.randn(batch, k, k, generator=gen, dtype=torch.float64, device=device) / math.sqrt(k)
    q1 = _orthonormal(gen, batch, k, k, device)
    q2 = _orthonormal(gen, batch, k, k, device)
    sig = decay ** torch.arange(k, dtype=torch.float64, device=device)
    return (q1 * sig) @ q2.transpose(1, 2)


def device_generator(tree: ClusterTree, k: int, seed: int = 0, decay=None, device=None) -> HbsFactorization:
    dev = torch.device(device) if device is not None else torch.device("cuda")
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    geo = tree_geometry(tree, k, dev)
    levels = [None] * (tree.depth + 1)
    for level in range(1, tree.depth + 1):
        g = geo[level]
        sizes = np.diff(g.begins_host)
        if level == tree.depth:
            uniq = np.unique(sizes)
            us, vs, ds = [], [], []
            if uniq.size == 1:
                m = int(uniq[0])
                u = _orthonormal(gen, g.nbox, m, k, dev).reshape(-1, k)
                v = _orthonormal(gen, g.nbox, m, k, dev).reshape(-1, k)
                d = torch.randn(g.nbox, m, m, generator=gen, dtype=torch.float64, device=dev) / math.sqrt(m)
                d += torch.eye(m, dtype=torch.float64, device=dev)
                levels[level] = (u.contiguous(), v.contiguous(), d.reshape(-1).contiguous())
            else:
                for m in sizes:
                    m = int(m)
                    us.append(_orthonormal(gen, 1, m, k, dev)[0])
                    vs.append(_orthonormal(gen, 1, m, k, dev)[0])
                    dd = torch.randn(m, m, generator=gen, dtype=torch.float64, device=dev) / math.sqrt(m)
                    ds.append((dd + torch.eye(m, dtype=torch.float64, device=dev)).reshape(-1))
                levels[level] = (torch.cat(us), torch.cat(vs), torch.cat(ds))
        else:
            u = _orthonormal(gen, g.nbox, 2 * k, k, dev).reshape(-1, k)
            v = _orthonormal(gen, g.nbox, 2 * k, k, dev).reshape(-1, k)
            d = torch.zeros(g.nbox, 2 * k, 2 * k, dtype=torch.float64, device=dev)
            d[:, :k, k:] = _coupling(gen, g.nbox, k, decay, dev)
            d[:, k:, :k] = _coupling(gen, g.nbox, k, decay, dev)
            levels[level] = (u.contiguous(), v.contiguous(), d.reshape(-1).contiguous())
    root = torch.zeros(2 * k, 2 * k, dtype=torch.float64, device=dev)
    root[:k, k:] = _coupling(gen, 1, k, decay, dev)[0]
    root[k:, :k] = _coupling(gen, 1, k, decay, dev)[0]
    return HbsFactorization.from_device(tree, k, geo, levels, root)


def device_samples(f: HbsFactorization, s: int, seed: int = 0):
    """Omega, Psi ~ N(0,1) (device Philox, seeded) and Y = A Omega, Z = A^T Psi
    through the device HBS sampler (hbs_apply)."""
    from .factorization import apply_matrix
    gen = torch.Generator(device=f.device)
    gen.manual_seed(seed + 1_000_003)
    om = torch.randn(f.n, s, generator=gen, dtype=torch.float64, device=f.device)
    ps = torch.randn(f.n, s, generator=gen, dtype=torch.float64, device=f.device)
    return om, ps, apply_matrix(f, om), apply_matrix(f, ps, transpose=True)


def _gen_level(gen, begins, k, leaf, decay, dev):
    """(U, V, D) packed for one level with row starts `begins` (numpy)."""
    sizes = np.diff(begins)
    nbox = sizes.size
    if not leaf:
        u = _orthonormal(gen, nbox, 2 * k, k, dev).reshape(-1, k)
        v = _orthonormal(gen, nbox, 2 * k, k, dev).reshape(-1, k)
        d = torch.zeros(nbox, 2 * k, 2 * k, dtype=torch.float64, device=dev)
        d[:, :k, k:] = _coupling(gen, nbox, k, decay, dev)
        d[:, k:, :k] = _coupling(gen, nbox, k, decay, dev)
        return u.contiguous(), v.contiguous(), d.reshape(-1).contiguous()
    us, vs, ds = [], [], []
    if (sizes == sizes[0]).all():
        m = int(sizes[0])
        u = _orthonormal(gen, nbox, m, k, dev).reshape(-1, k)
        v = _orthonormal(gen, nbox, m, k, dev).reshape(-1, k)
        d = torch.randn(nbox, m, m, generator=gen, dtype=torch.float64, device=dev) / math.sqrt(m)
        d += torch.eye(m, dtype=torch.float64, device=dev)
        return u.contiguous(), v.contiguous(), d.reshape(-1).contiguous()
    for m in sizes:
        m = int(m)
        us.append(_orthonormal(gen, 1, m, k, dev)[0])
        vs.append(_orthonormal(gen, 1, m, k, dev)[0])
        dd = torch.randn(m, m, generator=gen, dtype=torch.float64, device=dev) / math.sqrt(m)
        ds.append((dd + torch.eye(m, dtype=torch.float64, device=dev)).reshape(-1))
    return torch.cat(us), torch.cat(vs), torch.cat(ds)


def partitioned_generator(partition, k, seed=0, decay=None, device=None, group=None):
    """Exact-rank synthetic operator split by subtree (distributed.SubtreePartition):
    the rank's local levels from seed (seed, rank) and the replicated top
    levels + root from a seed shared by all ranks.  Returns a
    distributed.DistributedOperator (the multi-GPU sampler)."""
    from .distributed import DistributedOperator
    from .factorization import LevelGeometry
    dev = torch.device(device) if device is not None else torch.device("cuda")
    tree = partition.tree
    gl = torch.Generator(device=dev)
    gl.manual_seed(1_000_000 * (seed + 1) + partition.rank)
    local_blocks, local_geo = {}, {}
    for level, begins, _ in partition.local_specs:
        local_geo[level] = LevelGeometry(begins, dev)
        local_blocks[level] = _gen_level(gl, begins, k, level == tree.depth, decay, dev)
    gt = torch.Generator(device=dev)
    gt.manual_seed(seed)
    top_blocks, top_geo = {}, {}
    for level, begins, _ in partition.top_specs:
        top_geo[level] = LevelGeometry(begins, dev)
        top_blocks[level] = _gen_level(gt, begins, k, False, decay, dev)
    root = torch.zeros(2 * k, 2 * k, dtype=torch.float64, device=dev)
    root[:k, k:] = _coupling(gt, 1, k, decay, dev)[0]
    root[k:, :k] = _coupling(gt, 1, k, decay, dev)[0]
    return DistributedOperator(partition, local_blocks, local_geo, top_blocks, top_geo, root, group)
