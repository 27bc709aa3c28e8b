"""Run one c4-shaped level with the tracing library and print hqr phase cycles (CTA 0)."""
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
plan.run(om, ps, y, z); torch.cuda.synchronize()
# single level call for a clean trace of the leaf-level factor kernel
lib = nat.lib()
g = plan.geometry[tree.depth]
u, v, d = plan.levels[tree.depth]
out = plan.lift[0]
lib.hbs_compress_level(g.nbox, g.row_begin.data_ptr(), g.sq_off.data_ptr(), g.max_rows, 192, 64, 1e-10,
                       om.data_ptr(), ps.data_ptr(), y.data_ptr(), z.data_ptr(), u.data_ptr(), v.data_ptr(), d.data_ptr(),
                       *(m.data_ptr() for m in out), plan.workspace.data_ptr(), plan.workspace_bytes,
                       plan.status.data_ptr(), 0)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 320)()
getattr(lib, "hbs_debug_hqr_trace")(buf)
t = list(buf)
f = t[128:128 + 48]
print("FUSED (cycles from start):", {"P panel ready": [f[1 + 2 * p] - f[0] for p in range(4)],
      "P trailing done": [f[2 + 2 * p] - f[0] for p in range(4)], "P rinv done": f[20] - f[0],
      "Y panel done": [f[30 + p] - f[0] for p in range(4)], "Y solve start": f[40] - f[0], "Y end": f[41] - f[0]})
print("P per panel: start", [f[21 + 2 * p] - f[0] for p in range(4)], "pre-update done", [f[22 + 2 * p] - f[0] for p in range(4)],
      "factor done", [f[42 + p] - f[0] for p in range(4)])
sm = t[200:208]
print("STEP(j=6, panel 1, publisher): wait", sm[1]-sm[0], "loads+dots", sm[2]-sm[1], "reduce", sm[3]-sm[2], "updates until pub", sm[4]-sm[3], "norm+store", sm[5]-sm[4], "reflector", sm[6]-sm[5], "arrive", sm[7]-sm[6])
print("load", t[1] - t[0])
for p in range(4):
    a = 2 + 4 * p
    print(f"panel {p}: factor {t[a+1]-t[a]}  gram+T {t[a+2]-t[a+1]}  trailing {t[a+3]-t[a+2]}")
print("outputs", t[41] - t[40], "total", t[41] - t[0])
st = t[64:64 + 32]
print("step intervals (panel 0):", [st[i + 1] - st[i] for i in range(31)])
sp = t[64 + 40: 64 + 56]
for q in range(4):
    a = sp[4 * q: 4 * q + 4]
    print(f"sub {q}: end-of-steps->finalised {a[1]-a[0]}  W partial {a[2]-a[1]}  W'+update {a[3]-a[2]}  (steps start {st[8*q]-t[2]})")
pf = t[256:320]
base = f[0]
print("panel-factor per-warp marks (cycles from fused start; 0 start, 1 earlier reflectors applied, 2 first norm, 3..6 own steps):")
for w in range(8):
    print(f"  warp {w}:", [pf[8 * w + i] - base if pf[8 * w + i] else None for i in range(7)])
