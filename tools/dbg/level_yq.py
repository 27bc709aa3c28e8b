"""Debug: the fused kernel's YQ workspace for the first parent level vs numpy."""
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
ins = []
for idx in range(2):
    ins.append(quad)
    quad = plan.run_level(idx, quad, st)
    if not os.environ.get("NOSYNC"):
        torch.cuda.synchronize()
torch.cuda.synchronize()
for idx in range(1, 2):
    lifted_in = ins[idx]
    level = plan.specs[idx][0]
    g = plan.geometry[level]
    nr = g.max_rows
    ws = plan.workspace[: g.nbox * nr * s].view(g.nbox, nr, s).cpu().numpy()
    OM, Y = lifted_in[0].cpu().numpy(), lifted_in[2].cpu().numpy()
    ex, ep = 0.0, 0.0
    for b in range(g.nbox):
        rows = slice(int(g.begins_host[b]), int(g.begins_host[b + 1]))
        ob, yb = OM[rows], Y[rows]
        q = np.linalg.qr(ob.T, mode="complete")[0]
        yq = yb @ q
        nb = ob.shape[0]
        xr = yb @ np.linalg.pinv(ob)
        ex = max(ex, np.abs(ws[b, :nb, :nb] - xr).max() / np.abs(xr).max())
        ep = max(ep, np.abs(ws[b, :nb, s - r:] - yq[:, s - r:]).max() / np.abs(yq[:, s - r:]).max())
    print(f"level {level}: X rel err {ex:.2e}  YP rel err {ep:.2e}")
