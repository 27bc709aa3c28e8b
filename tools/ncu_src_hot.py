"""Hottest CUDA source lines (warp-stall samples) of a kernel in an ncu report:
python tools/ncu_src_hot.py rep.ncu-rep [kernel-regex] [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if kern:
    cmd += ["-k", "regex:" + kern]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
agg = collections.Counter()
src = {}
fname = None
hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < 5:
        continue
    try:
        line = int(row[0])
        samples = int(row[4] or 0)
    except ValueError:
        continue
    agg[(fname, line)] += samples
    src[(fname, line)] = row[1][:90]
total = sum(agg.values()) or 1
for (f, l), v in agg.most_common(top):
    print(f"{100.0 * v / total:5.1f}%  {f}:{l:<5d} {src[(f, l)]}")
