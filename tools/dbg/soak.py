"""Soak: many sweeps (graph replays and stream launches) of c4-shaped trees; every result must hash the same."""
import hashlib, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch
import paper_2205_02990_b200 as hb
from paper_2205_02990_b200 import synthetic
def digest(plan):
    h = hashlib.sha256()
    for level in sorted(plan.levels):
        for m in plan.levels[level]:
            h.update(m.cpu().numpy().tobytes())
    h.update(plan.root.cpu().numpy().tobytes())
    return h.hexdigest()
for n, reps in ((1 << 14, 400), (1 << 17, 200), (1000000, 20), (1 << 20, 20)):
    tree = hb.build_tree(n, 128)
    gen = synthetic.device_generator(tree, 64, seed=0, decay=0.9)
    quad = synthetic.device_samples(gen, 192)
    del gen
    plan = hb.CompressPlan(tree, 192, 64)
    plan.run(*quad); torch.cuda.synchronize(); plan.raise_for_status()
    want = digest(plan)
    bad = 0
    for i in range(reps):
        if i % 2:
            plan.run(*quad)
        else:
            plan.run_graph(*quad)
        if i % max(1, reps // 8) == 0 or i == reps - 1:
            torch.cuda.synchronize(); plan.raise_for_status()
            bad += digest(plan) != want
    torch.cuda.synchronize()
    print(f"N={n}: {reps} sweeps, mismatching digests: {bad}", flush=True)
    del plan, quad
    torch.cuda.empty_cache()
