import sys, numpy as np
a = np.loadtxt(sys.argv[1], dtype=np.int64)
names = ["tma_issue", "split_full", "split_done", "mma_start", "mma_issued", "epi_full", "epiP_done", "epiQ_done",
         "e_ld0", "e_math0", "e_shfl0", "e_bar_out", "e_bar_in", "x", "y", "z"]
t0 = a[0][0]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
print("tile " + " ".join(f"{x:>10}" for x in names[:13]))
for i in range(n):
    print(f"{i:4d} " + " ".join(f"{(a[k][i]-t0) if a[k][i] else -1:>10d}" for k in range(13)))
d = lambda k: np.diff(a[k][a[k] > 0])
for k in range(8):
    v = d(k)
    if len(v): print(f"{names[k]:>12}: median step {np.median(v):.0f} cyc")
