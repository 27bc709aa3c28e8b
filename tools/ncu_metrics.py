"""Print selected raw metrics of the first kernel in an ncu report: python tools/ncu_metrics.py rep substr..."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units, v = rows[0], rows[1], rows[2]
for k, u, x in zip(h, units, v):
    if any(s in k for s in sys.argv[2:]):
        print(f"{k:90s} {x} {u}")
