"""Debug: lifted quadruple of the leaf level vs the oracle's lift."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np, torch
import paper_2205_02990_b200 as hb
from oracle import hbs_oracle as O
n, leaf, r, s = 256, 16, 8, 48
rng = np.random.default_rng(77)
a = rng.standard_normal((n, n)) / np.sqrt(n)
om, ps = O.gaussian(n, s, 5, 0), O.gaussian(n, s, 5, 1)
y, z = a @ om, a.T @ ps
tree = hb.build_tree(n, leaf)
plan = hb.CompressPlan(tree, s, r)
dev = torch.device("cuda")
quad = tuple(torch.from_numpy(m).to(dev) for m in (om, ps, y, z))
st = torch.cuda.current_stream().cuda_stream
out = plan.run_level(0, quad, st)
torch.cuda.synchronize()
u, v, d = (t.cpu().numpy() for t in plan.levels[tree.depth])
lifted = [t.cpu().numpy() for t in out]
g = plan.geometry[tree.depth]
errs = np.zeros(4)
for b in range(g.nbox):
    rows = slice(int(g.begins_host[b]), int(g.begins_host[b + 1]))
    nb = rows.stop - rows.start
    ub, vb = u[rows], v[rows]
    db = d[int(g.sq_host[b]): int(g.sq_host[b + 1])].reshape(nb, nb)
    ref = O.lift_rows(ub, vb, db, om[rows], ps[rows], y[rows], z[rows])
    for i in range(4):
        got = lifted[i][b * r:(b + 1) * r]
        errs[i] = max(errs[i], np.abs(got - ref[i]).max() / np.abs(ref[i]).max())
print("lift rel err (omega, psi, y, z):", errs)
