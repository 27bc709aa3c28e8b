"""Clock64 phase trace of the TMEM Gram kernel's first CTA (HBS_TRACE build,
tools/variants/hbs_trace.so) at the root level (runs alone)."""
import ctypes, os, sys
os.environ.setdefault("HBS_B200_LIB", os.path.join(os.path.dirname(__file__), "..", "variants", "hbs_trace.so"))
os.environ["HBS_GRAM"] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch
import paper_2205_02990_b200 as hb
from paper_2205_02990_b200 import synthetic, _native
lib = _native.lib()
lib.hbs_debug_gram_tm_trace.argtypes = [ctypes.c_void_p]
n = int(os.environ.get("N", 1 << 14))
tree = hb.build_tree(n, 128)
gen = synthetic.device_generator(tree, 64, seed=0, decay=0.9)
om, ps, y, z = synthetic.device_samples(gen, 192)
plan = hb.CompressPlan(tree, 192, 64)
plan.run(om, ps, y, z)
torch.cuda.synchronize()
b = (ctypes.c_longlong * 32)()
lib.hbs_debug_gram_tm_trace(b)
t0 = b[0]
print("total", b[9] - t0, " G", b[1] - t0, " LU loop", b[7] - b[1], " screen", b[8] - b[7], " V2", b[9] - b[8])
print("iteration 3: A", b[3] - b[2], " B", b[4] - b[3], " B2", b[5] - b[4], " C", b[6] - b[5])
