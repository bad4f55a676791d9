"""Top SASS instructions by warp-stall samples, with a few preceding instructions as context (dev tool).
usage: python tools/ncu_sass_hot.py report.ncu-rep [topN] [context]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 3
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = None
ins = []
for r in rows:
    if r and r[0] == "Address":
        h = r
        si = h.index("Warp Stall Sampling (All Samples)")
        ie = h.index("Instructions Executed")
        continue
    if h is None or len(r) <= si:
        continue
    try:
        ins.append((r[0], r[1].strip(), int(r[si] or 0), int(r[ie] or 0)))
    except ValueError:
        pass
tot = sum(x[2] for x in ins)
order = sorted(range(len(ins)), key=lambda i: -ins[i][2])[:top]
print("total samples", tot)
for i in order:
    a, s, n, e = ins[i]
    print(f"{n:6d} {100*n/tot:5.1f}%  ex {e:9d}  {a[-5:]}  {s}")
    for j in range(max(0, i - ctx), i):
        print(f"{'':30s}{ins[j][0][-5:]}  {ins[j][1][:100]}")
