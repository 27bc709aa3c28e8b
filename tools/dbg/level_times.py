"""Per-level device time of the c4 sweep (CUDA events around each level)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch
import paper_2205_02990_b200 as hb
from paper_2205_02990_b200 import synthetic
n = int(os.environ.get("N", 1 << 20))
tree = hb.build_tree(n, 128)
gen = synthetic.device_generator(tree, 64, seed=0, decay=0.9)
om, ps, y, z = synthetic.device_samples(gen, 192)
plan = hb.CompressPlan(tree, 192, 64)
st = torch.cuda.current_stream().cuda_stream
for rep in range(2):
    quad = (om, ps, y, z)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(plan.specs) + 2)]
    ev[0].record()
    for idx in range(len(plan.specs)):
        quad = plan.run_level(idx, quad, st)
        ev[idx + 1].record()
    plan.run_root(quad[0], quad[2])
    ev[-1].record()
    torch.cuda.synchronize()
out = [f"L{plan.specs[i][0]}:{ev[i].elapsed_time(ev[i + 1]):.2f}" for i in range(len(plan.specs))]
print("ms per level:", " ".join(out), f"root:{ev[-2].elapsed_time(ev[-1]):.2f}", f"total:{ev[0].elapsed_time(ev[-1]):.2f}")
