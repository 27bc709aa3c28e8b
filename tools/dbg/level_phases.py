"""Per-level phase times (hbs_compress_level_profiled) of the c4 sweep."""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch
import paper_2205_02990_b200 as hb
from paper_2205_02990_b200 import synthetic, _native
n = int(os.environ.get("N", 1 << 20))
tree = hb.build_tree(n, 128)
gen = synthetic.device_generator(tree, 64, seed=0, decay=0.9)
om, ps, y, z = synthetic.device_samples(gen, 192)
plan = hb.CompressPlan(tree, 192, 64)
plan.run(om, ps, y, z); torch.cuda.synchronize()
lib = _native.lib()
st = torch.cuda.current_stream().cuda_stream
buf = (ctypes.c_float * 6)()
quad = (om, ps, y, z)
for idx, level in enumerate(range(tree.depth, 0, -1)):
    g = plan.geometry[level]
    u, v, d = plan.levels[level]
    out = plan.lift[idx % 2]
    _native.check(lib.hbs_compress_level_profiled(g.nbox, g.row_begin.data_ptr(), g.sq_off.data_ptr(), g.max_rows, 192, 64,
                  plan.tol, *(m.data_ptr() for m in quad), u.data_ptr(), v.data_ptr(), d.data_ptr(),
                  *(m.data_ptr() for m in out), plan.workspace.data_ptr(), plan.workspace_bytes, plan.status.data_ptr(),
                  st, buf), "profiled")
    quad = tuple(m[:g.nbox * 64] for m in out)
    print(f"L{level:2d} nbox {g.nbox:5d}  probe {buf[0]:7.3f} {buf[1]:7.3f} {buf[2]:7.3f}  basis {buf[3]:6.3f}  disc {buf[4]:6.3f}  lift {buf[5]:6.3f} ms")
