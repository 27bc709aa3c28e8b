"""Summarise an ncu source page (CSV) by hottest lines: python tools/ncu_hot.py rep.ncu-rep [kernel-regex] [cuda|sass]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else None
mode = sys.argv[3] if len(sys.argv) > 3 else "cuda"
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", mode]
if kern:
    cmd += ["-k", "regex:" + kern]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name"')
for blk in blocks[1:2]:
    lines = blk.splitlines()
    print("Kernel", lines[0][:120])
    rdr = csv.reader(io.StringIO("\n".join(lines[1:])))
    hdr = next(rdr)
    rows = [r for r in rdr if len(r) == len(hdr)]
    i_src = hdr.index("Source")
    i_st = hdr.index("Warp Stall Sampling (All Samples)")
    i_ex = hdr.index("Instructions Executed")
    tot_st = sum(float(r[i_st] or 0) for r in rows)
    tot_ex = sum(float(r[i_ex] or 0) for r in rows)
    print(f"total stall samples {tot_st:.0f}, instructions {tot_ex:.3e}")
    rows.sort(key=lambda r: -float(r[i_st] or 0))
    for r in rows[:25]:
        print(f"{100*float(r[i_st] or 0)/tot_st:5.1f}% st {100*float(r[i_ex] or 0)/tot_ex:5.1f}% ex | {r[i_src].strip()[:110]}")

# opcode histogram by executed instructions (first kernel)
import collections
hist = collections.Counter()
for r in rows:
    op = r[i_src].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1] if len(op) > 1 else o
    hist[o.split(".")[0]] += float(r[i_ex] or 0)
print("opcode mix:", ", ".join(f"{k} {100*v/tot_ex:.1f}%" for k, v in hist.most_common(18)))
