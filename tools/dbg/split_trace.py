"""Clock64 trace of the SMSP-split pipelined kernel (HBS_TRACE build, tools/variants/hbs_trace.so):
second item of CTA 0 (steady state) at the leaf level of a c4-shaped tree."""
import ctypes, os, sys
os.environ["HBS_SPLIT"] = "1"
os.environ.setdefault("HBS_B200_LIB", os.path.join(os.path.dirname(__file__), "..", "variants", "hbs_trace.so"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch
import paper_2205_02990_b200 as hb
from paper_2205_02990_b200 import synthetic, _native
lib = _native.lib()
n = int(os.environ.get("N", 1 << 17))
tree = hb.build_tree(n, 128)
gen = synthetic.device_generator(tree, 64, seed=0, decay=0.9)
om, ps, y, z = synthetic.device_samples(gen, 192)
plan = hb.CompressPlan(tree, 192, 64)
g = plan.geometry[tree.depth]
u, v, d = plan.levels[tree.depth]
out = plan.lift[0]
for _ in range(2):
    lib.hbs_compress_level(g.nbox, g.row_begin.data_ptr(), g.sq_off.data_ptr(), g.max_rows, 192, 64, 1e-10,
                           om.data_ptr(), ps.data_ptr(), y.data_ptr(), z.data_ptr(), u.data_ptr(), v.data_ptr(), d.data_ptr(),
                           *(m.data_ptr() for m in out), plan.workspace.data_ptr(), plan.workspace_bytes,
                           plan.status.data_ptr(), 0)
    torch.cuda.synchronize()
b = (ctypes.c_longlong * 96)()
lib.hbs_debug_split_trace.argtypes = [ctypes.c_void_p]
lib.hbs_debug_split_trace(b)
t = list(b)
t0 = t[0]
for k in range(3):
    r = lambda i: t[32 * k + i] - t0
    print(f"--- item {k + 1} of CTA 0 (cycles from item 1's panel-0 landing)")
    print("P: panel-0 columns landed", r(0), " p0 factor start", r(1), " p0 ready", r(8), " ydone(prev) seen", r(13))
    for p in (1, 2, 3):
        print(f"P: panel {p}: waits done {r(2*p)}  look-ahead done {r(2*p+1)}  ready {r(8+p)}")
    print("P: last rinv done", r(12))
    print("Y: rows in TMEM", r(16), " panel done", [r(17 + p) for p in range(4)], " solve done / ydone", r(21), " written back", r(22))
