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
