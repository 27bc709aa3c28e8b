"""Per-CUDA-source-line stall / instruction attribution from an ncu report.
usage: python tools/ncu_lines.py rep.ncu-rep kernel-regex [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      "regex:" + kern], capture_output=True, text=True).stdout
rows, fname, func, seen_funcs = [], None, None, []
sel = sys.argv[4] if len(sys.argv) > 4 else ""
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] == "Function Name":
        func = rec[1]
        if func not in seen_funcs:
            seen_funcs.append(func)
        continue
    if rec[0] == "Line No" or not func or not (sel in func):
        continue
    if rec[0] and rec[2] == "-":
        try:
            rows.append((fname, int(rec[0]), rec[1].strip(), float(rec[4]), float(rec[7])))
        except ValueError:
            pass
tot_s = sum(r[3] for r in rows) or 1
tot_i = sum(r[4] for r in rows) or 1
print("kernels:", [f[:60] for f in seen_funcs], "selected:", sel)
for r in sorted(rows, key=lambda r: -r[3])[:top]:
    print(f"{100*r[3]/tot_s:5.1f}% stall {100*r[4]/tot_i:5.1f}% inst  {r[0]}:{r[1]}  {r[2][:90]}")
