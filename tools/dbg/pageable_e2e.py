"""Time compress_from_samples with ordinary (pageable) numpy inputs at config 4 (N from env)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import numpy as np, torch
import paper_2205_02990_b200 as hb
from paper_2205_02990_b200 import synthetic
n = int(os.environ.get("N", 1 << 20))
tree = hb.build_tree(n, 128)
gen = synthetic.device_generator(tree, 64, seed=0, decay=0.9)
quad = [m.cpu().numpy() for m in synthetic.device_samples(gen, 192)]
del gen
torch.cuda.empty_cache()
cfg = hb.CompressionConfig(rank=64, leaf_threshold=128)
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    f = hb.compress_from_samples(hb.SampleSet(*quad), tree, cfg)
    f.materialize()
    print("pageable call", it, round(time.perf_counter() - t0, 4), "s", flush=True)
    del f
t0 = time.perf_counter()
a = torch.empty(n // 16, 192, dtype=torch.float64, pin_memory=True)
print("pinned alloc 100 MB", round(time.perf_counter() - t0, 4))
src = torch.from_numpy(quad[0])
t0 = time.perf_counter()
for k in range(16):
    a.copy_(src[k * (n // 16):(k + 1) * (n // 16)])
print("16 host copies of 100 MB:", round(time.perf_counter() - t0, 4), "s; torch threads", torch.get_num_threads())
