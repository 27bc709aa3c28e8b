"""Checksums (sha256 of the raw bytes) of one c4-shaped sweep's U, V, D and root at N
(env N, default 2^17), for bitwise A/B comparisons of kernel variants."""
import hashlib, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch
import paper_2205_02990_b200 as hb
from paper_2205_02990_b200 import synthetic
n = int(os.environ.get("N", 1 << 17))
tree = hb.build_tree(n, 128)
gen = synthetic.device_generator(tree, 64, seed=0, decay=0.9)
om, ps, y, z = synthetic.device_samples(gen, 192)
plan = hb.CompressPlan(tree, 192, 64)
for rep in range(int(os.environ.get("REPS", 2))):
    plan.run(om, ps, y, z)
    torch.cuda.synchronize()
    plan.raise_for_status()
    h = hashlib.sha256()
    for level in sorted(plan.levels):
        for m in plan.levels[level]:
            h.update(m.cpu().numpy().tobytes())
    h.update(plan.root.cpu().numpy().tobytes())
    print("rep", rep, h.hexdigest())
