"""Per-SASS-instruction stall attribution from an ncu report (source page).
usage: python tools/ncu_sass_stalls.py rep.ncu-rep kernel-regex [top]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
rd = csv.reader(io.StringIO(out))
hdr, rows = None, []
for rec in rd:
    if len(rec) > 3 and rec[0] == "Address":
        hdr = rec
        continue
    if hdr and len(rec) == len(hdr):
        rows.append(dict(zip(hdr, rec)))
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
for r in rows:
    for h in reasons:
        tot[h] += float(r[h] or 0)
allsamp = sum(tot.values()) or 1
print("total samples", allsamp)
print("  ".join(f"{k[6:]} {100 * v / allsamp:.1f}%" for k, v in tot.most_common(10)))
rows.sort(key=lambda r: -float(r["Warp Stall Sampling (All Samples)"] or 0))
for r in rows[:top]:
    s = float(r["Warp Stall Sampling (All Samples)"] or 0)
    c = Counter({h[6:]: float(r[h] or 0) for h in reasons})
    print(f"{r['Address'][-5:]} {100 * s / allsamp:5.2f}% {r['Source'].strip()[:60]:60s} " +
          " ".join(f"{k}:{int(v)}" for k, v in c.most_common(3) if v))
