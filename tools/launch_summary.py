"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"].split("(")[0][:70]
            v = float(d["Metric Value"].replace(",", "")) * scale.get(d.get("Metric Unit", "nsecond"), 1e-3)
            agg[k][0] += 1
            agg[k][1] += v
tot = sum(v[1] for v in agg.values())
print("%6s %12s %8s %6s  %s" % ("count", "total_us", "avg_us", "share", "kernel"))
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print("%6d %12.1f %8.1f %5.1f%%  %s" % (n, t, t / n, 100 * t / tot, k))
