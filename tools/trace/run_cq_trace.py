"""Run one c4-shaped level with the tracing library and print the CholeskyQR2 phase cycles (CTA 0)."""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import paper_2205_02990_b200._native as nat
nat.LIB_PATH = os.environ.get("HBS_B200_LIB") or os.path.join(os.path.dirname(__file__), "_hbs_b200_trace.so")
import torch
import paper_2205_02990_b200 as hb
from paper_2205_02990_b200 import synthetic
tree = hb.build_tree(1 << 14, 128)
gen = synthetic.device_generator(tree, 64, seed=0, decay=0.9)
om, ps, y, z = synthetic.device_samples(gen, 192)
plan = hb.CompressPlan(tree, 192, 64)
plan.run_level(0, (om, ps, y, z), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 32)()
nat.lib().hbs_debug_cq_trace(buf)
t = list(buf)
names = {0: "start", 1: "loaded", 2: "gram1", 8: "chol blk0", 9: "chol blk1", 10: "chol blk2", 11: "chol blk3",
         12: "chol done", 13: "trinv", 14: "apply R^-1", 5: "gram2", 15: "e-check+polar B", 16: "apply B"}
prev = t[0]
for i in [1, 2, 8, 9, 10, 11, 12, 13, 14, 5, 15, 16]:
    print(f"{names[i]:18s} +{t[i] - prev:7d}  (at {t[i] - t[0]})")
    prev = t[i]
