"""One compress sweep at the c4 shape (N from env, default 2^16) -- for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch
import paper_2205_02990_b200 as hb
from paper_2205_02990_b200 import synthetic
n = int(os.environ.get("N", 1 << 16))
tree = hb.build_tree(n, 128)
gen = synthetic.device_generator(tree, 64, seed=0, decay=0.9)
om, ps, y, z = synthetic.device_samples(gen, 192)
plan = hb.CompressPlan(tree, 192, 64)
for _ in range(int(os.environ.get("REPS", 2))):
    plan.run(om, ps, y, z)
torch.cuda.synchronize()
print("ok")
