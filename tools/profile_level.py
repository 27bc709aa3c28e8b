"""Small c4-shaped compress (N = 2^16 by default) for ncu captures."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2205_02990_b200 as hb
from paper_2205_02990_b200 import synthetic

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 16)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--leaf", type=int, default=128)
ap.add_argument("--s", type=int, default=192)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
tree = hb.build_tree(a.n, a.leaf)
gen = synthetic.device_generator(tree, a.k, seed=0, decay=0.9)
om, ps, y, z = synthetic.device_samples(gen, a.s)
plan = hb.CompressPlan(tree, a.s, a.k)
for _ in range(a.reps):
    plan.run(om, ps, y, z)
torch.cuda.synchronize()
plan.raise_for_status()
print("ok")
