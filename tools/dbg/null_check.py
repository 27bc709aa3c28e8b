"""Debug: per-level projector agreement with the oracle for nullity > r cases."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np
import paper_2205_02990_b200 as hb
from oracle import hbs_oracle as O
for (n, leaf, r, s) in [(256, 16, 8, 48)]:
    rng = np.random.default_rng(77)
    a = rng.standard_normal((n, n)) / np.sqrt(n)
    om, ps = O.gaussian(n, s, 5, 0), O.gaussian(n, s, 5, 1)
    y, z = a @ om, a.T @ ps
    tree = hb.build_tree(n, leaf)
    import torch
    dev = os.environ.get("DEV_INPUT")
    smp = hb.SampleSet(*(torch.from_numpy(m).cuda() for m in (om, ps, y, z))) if dev else hb.SampleSet(om, ps, y, z)
    f = hb.compress_from_samples(smp, tree, hb.CompressionConfig(rank=r, leaf_threshold=leaf))
    ref = O.compress(om, ps, y, z, O.level_bounds(n, tree.depth), r)
    out = []
    for level in range(tree.depth, 0, -1):
        e = max(np.linalg.norm(f.u_bases[(1 << level) - 1 + j] @ f.u_bases[(1 << level) - 1 + j].T - ref.U[level][j] @ ref.U[level][j].T) for j in range(1 << level))
        ev = max(np.linalg.norm(f.v_bases[(1 << level) - 1 + j] @ f.v_bases[(1 << level) - 1 + j].T - ref.V[level][j] @ ref.V[level][j].T) for j in range(1 << level))
        ed = max(np.linalg.norm(f.discs[(1 << level) - 1 + j] - ref.D[level][j]) for j in range(1 << level))
        out.append(f"L{level}(rows {ref.U[level][0].shape[0]}): U {e:.1e} V {ev:.1e} D {ed:.1e}")
    print((n, leaf, r, s), " ".join(out))
