"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) per kernel:
python scripts/launch_summary.py launches.csv out.csv"""
import collections, csv, re, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
agg = collections.OrderedDict()
for r in rows[hdr + 1:]:
    d = dict(zip(rows[hdr], r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("<unnamed>::", "")
    v = float(d["Metric Value"].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(d["Metric Unit"], 1e-6)
    agg.setdefault(name, []).append(v)
total = sum(sum(v) for v in agg.values())
with open(sys.argv[2], "w", newline="") as fh:
    wr = csv.writer(fh)
    wr.writerow(["kernel", "launches", "total_ms", "mean_ms", "share"])
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        wr.writerow([k, len(v), f"{sum(v):.3f}", f"{sum(v) / len(v):.3f}", f"{sum(v) / total:.4f}"])
print(open(sys.argv[2]).read())
