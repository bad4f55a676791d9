"""Aggregate ncu warp-stall samples by CUDA source line (dev tool).
usage: python tools/ncu_src.py report.ncu-rep [topN]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
data = []
h = None
for r in rows:
    if r and r[0] == "Line No":
        h = r
        si = h.index("Warp Stall Sampling (All Samples)")
        ni = h.index("Warp Stall Sampling (Not-issued Samples)")
        ie = h.index("Instructions Executed")
        continue
    if h is None or len(r) <= si or r[2] != "-":
        continue  # keep the per-source-line aggregate rows (Address == "-")
    try:
        data.append((int(r[si]), int(r[ni]), int(r[ie]), r[0], r[1].strip()))
    except ValueError:
        pass
tot = sum(d[0] for d in data)
print("total samples", tot)
for d in sorted(data, reverse=True)[:top]:
    print(f"{d[0]:7d} {100*d[0]/max(tot,1):5.1f}% (ni {d[1]:6d}) ex {d[2]:9d} L{d[3]:>5}  {d[4][:100]}")
