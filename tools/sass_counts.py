"""Per-kernel SASS instruction counts of libkrp.so (static): python tools/sass_counts.py [lib]
UTCHMMA = tcgen05.mma, UTMALDG = TMA tensor load, UBLKCP = bulk copy, LDTM / STTM = tcgen05.ld / st,
DMMA = fp64 tensor-core mma.sync, USETMAXREG = setmaxnreg, SYNCS = mbarrier ops, STL / LDL = local spills."""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2507_23207_b200/libkrp.so"
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout.split("\n")
keys = ["UTCHMMA", "UTMALDG", "UBLKCP", "LDTM", "STTM", "DMMA", "USETMAXREG", "SYNCS", "STL", "LDL"]
fn, cnt = None, {}
for line in txt:
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1)
        cnt[fn] = {k: 0 for k in keys}
        continue
    if fn:
        for k in keys:
            if re.search(r"\b" + k, line):
                cnt[fn][k] += 1


def short(n):
    m = re.search(r"krp_tc_sketch_kernelILi(\d+)ELi(\d+)", n)
    if m:
        return f"krp_tc_sketch_kernel<{m.group(1)},{m.group(2)}>"
    m = re.search(r"ttm0_tc_kernelILb(\d)", n)
    if m:
        return f"ttm0_tc_kernel<{m.group(1)}>"
    m = re.search(r"_cu_\w+?\d+([a-z_0-9]+_kernel)", n)
    return m.group(1) if m else n[:40]


print(f"{'kernel':44s}" + "".join(f"{k:>11s}" for k in keys))
for n, c in cnt.items():
    print(f"{short(n):44s}" + "".join(f"{c[k]:>11d}" for k in keys))
