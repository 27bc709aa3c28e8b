"""Generates pfq_trace.inc: panel_factor_q from hqr.cu with per-step clock
stamps in the publishing lane (development tool for panel_bench.cu)."""
import re

src = open('/root/repo/paper_2205_02990_b200/csrc/hqr.cu').read()
a = src.index("template <int MR8, int NTG>\nHBS_DEV void panel_factor_q(")
e = src.index("// G = V_p^T V_p (32 x 32)")
f = src[a:e].replace("panel_factor_q(", "pfq_trace(").replace(
    "double* G, double* s_an) {", "double* G, double* s_an, long long* trc) {\n  double* Tscr_sink = s_beta + 63;")
f = re.sub(r"const bool tr = [^\n]*", "const bool rec = own && (q == j + 1) && li == 0 && blockIdx.x == 0;\n        double* sink = Tscr_sink;", f)


def ins(k, dep):
    global f
    tag = f"if (tr) STEP_MARK({k});"
    assert tag in f, tag
    dep_st = (f"asm volatile(\"st.volatile.shared.f64 [%0], %1;\" :: \"r\"((unsigned)__cvta_generic_to_shared(sink)), "
              f"\"d\"({dep}) : \"memory\"); ") if dep else ""
    f = f.replace(tag, f"if (rec) {{ {dep_st}trc[j * 10 + {k}] = clock64(); }}")


for k, dep in [(0, "0.0"), (1, "tau*scale"), (2, "pv[0]+pv[MR8-1]"), (3, "dd[0]+dd[7]"), (4, "d"),
               (5, "x[0]+x[MR8-1]"), (6, "nrm+alpha"), (7, "nrm"), (8, None), (9, None)]:
    ins(k, dep)
open('/root/repo/tools/micro/pfq_trace.inc', 'w').write("namespace hbs {\n" + f + "}\n")
