"""Clock64 phase trace of the Gram kernel's first CTA (HBS_TRACE build in
tools/variants/hbs_trace.so): start, after G, after Cholesky, after LU, end."""
import ctypes, os, sys
os.environ.setdefault("HBS_B200_LIB", os.path.join(os.path.dirname(__file__), "..", "variants", "hbs_trace.so"))
os.environ["HBS_GRAM"] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch
import paper_2205_02990_b200 as hb
from paper_2205_02990_b200 import synthetic, _native
lib = _native.lib()
lib.hbs_debug_gram_trace.argtypes = [ctypes.c_void_p]
n = int(os.environ.get("N", 1 << 14))
tree = hb.build_tree(n, 128)
gen = synthetic.device_generator(tree, 64, seed=0, decay=0.9)
om, ps, y, z = synthetic.device_samples(gen, 192)
plan = hb.CompressPlan(tree, 192, 64)
plan.run(om, ps, y, z)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 32)()
lib.hbs_debug_gram_trace(buf)
t = [buf[i] - buf[0] for i in range(5)]
names = ["G", "Chol+LU to it=nb-1", "last LU it+screen", "V2/T/fac"]
print("root-level CTA (runs alone): total %d cycles" % t[4])
for i in range(4):
    print(f"  {names[i]:10s} {t[i + 1] - t[i]:8d} cycles")
it1_end, a, b_, c_ = buf[8], buf[5], buf[6], buf[7]
print(f"  iteration 2: A (diag chol/LU + inverses) {a - it1_end}  B (panels) {b_ - a}  C (trailing) {c_ - b_}")
print(f"  tail: V2/T {buf[9] - buf[3]}  R_hh/V1 rows {buf[4] - buf[9]}")
