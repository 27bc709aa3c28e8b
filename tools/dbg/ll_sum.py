"""Sum an ncu --csv launch list (gpu__time_duration.sum) by kernel: python tools/dbg/ll_sum.py file.csv"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            agg[d["Kernel Name"][:64]][0] += 1
            agg[d["Kernel Name"][:64]][1] += float(d["Metric Value"])
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"{v[1] / 1e6:9.3f} ms {v[0]:5d}  {k}")
print(f"{tot / 1e6:9.3f} ms total")
