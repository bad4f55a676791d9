"""Summarise one gpu_round.sh output directory into a committed text file under profiles/ (dev tool).

usage: python tools/ncu_summary.py gpurun_out/<tag> profiles/<tag>_summary.txt
Reads launches.csv (ncu --metrics gpu__time_duration.sum launch list), sketch_full.ncu-rep (ncu --set full
of the fused sketch kernel) and bench.log, and writes: the bench JSON line, per-kernel launch times and
their share of the step, and the counters DESIGN.md cites (DRAM bytes, tensor pipe, issue, stalls)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

src, dst = sys.argv[1], sys.argv[2]
out = []

bench = os.path.join(src, "bench.log")
if os.path.exists(bench):
    for line in open(bench):
        if line.startswith("{"):
            out.append("bench: " + line.strip())

lc = os.path.join(src, "launches.csv")
if os.path.exists(lc):
    rows = list(csv.reader(open(lc)))
    h = None
    agg = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            h = r
            continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                unit = d.get("Metric Unit", "ns")
                v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
                nm = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
                a = agg.setdefault(nm, [0, 0.0])
                a[0] += 1
                a[1] += v
    tot = sum(a[1] for a in agg.values())
    out.append("\nncu launch list (gpu__time_duration.sum, --clock-control none, cold cache, serialised):")
    out.append(f"{'launches':>8} {'avg us':>10} {'share':>7}  kernel")
    for nm, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{c:8d} {t / c:10.2f} {100 * t / tot:6.1f}%  {nm}")

rep = os.path.join(src, "sketch_full.ncu-rep")
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) >= 3:
        h, u = rows[0], rows[1]
        want = ["Kernel Name", "gpu__time_duration.sum", "gpc__cycles_elapsed.max.per_second", "dram__bytes_read.sum",
                "dram__bytes_write.sum", "dram__bytes_read.sum.per_second",
                "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
                "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
                "launch__block_size"]
        stalls = [k for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
        for r in rows[2:]:
            d = dict(zip(h, r))
            out.append("\nncu --set full capture of one launch:")
            for k in want:
                if k in d:
                    out.append(f"  {k} = {d[k]} {u[h.index(k)]}")
            st = sorted(((float(d[k] or 0), k) for k in stalls), reverse=True)[:8]
            out.append("  top stall reasons (warps per issue): " + ", ".join(
                f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
                for v, k in st))
    src_txt = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "ncu_src.py"), rep, "20"],
                             capture_output=True, text=True).stdout
    out.append("\nwarp-state samples by source line (top 20):\n" + src_txt)

with open(dst, "w") as f:
    f.write("\n".join(out) + "\n")
print("\n".join(out))
