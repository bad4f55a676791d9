"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: the last call's launches
(everything after the given number of leading launches), grouped by kernel.
python tools/launch_summary.py launches.csv [skip]"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hdr, out = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append((d["Kernel Name"].split("(")[0].replace("krp::<unnamed>::", ""), float(d["Metric Value"]) / 1e3))
out = out[skip:]
g = OrderedDict()
for k, us in out:
    c, t = g.get(k, (0, 0.0))
    g[k] = (c + 1, t + us)
tot = sum(t for _, t in g.values())
print(f"{len(out)} launches, {tot:.1f} us total")
for k, (c, t) in sorted(g.items(), key=lambda kv: -kv[1][1]):
    print(f"{c:5d} {t:10.1f} us {100 * t / tot:5.1f}%  {k}")
