"""Instruction / stall share by source-line ranges: python tools/ncu_regions.py rep kernel-regex select file a-b:name ..."""
import csv, io, subprocess, sys
rep, kern, sel = sys.argv[1], sys.argv[2], sys.argv[3]
ranges = []
for spec in sys.argv[4:]:
    f, rest = spec.split(":", 1)
    ab, name = rest.split("=")
    a, b = ab.split("-")
    ranges.append((f, int(a), int(b), name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
fname = func = None
acc = {r[3]: [0.0, 0.0] for r in ranges}
acc["other"] = [0.0, 0.0]
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]; continue
    if rec[0] == "Function Name":
        func = rec[1]; continue
    if rec[0] == "Line No" or not func or sel not in func:
        continue
    if rec[0] and rec[2] == "-":
        try:
            ln, st, ins = int(rec[0]), float(rec[4]), float(rec[7])
        except ValueError:
            continue
        key = "other"
        for f, a, b, name in ranges:
            if fname == f and a <= ln <= b:
                key = name
                break
        acc[key][0] += st
        acc[key][1] += ins
ts = sum(v[0] for v in acc.values()) or 1
ti = sum(v[1] for v in acc.values()) or 1
for k, v in acc.items():
    print(f"{k:20s} stall {100*v[0]/ts:5.1f}%  inst {100*v[1]/ti:5.1f}%  ({v[1]:.3e} inst)")
