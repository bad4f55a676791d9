import sys, numpy as np
a = np.loadtxt(sys.argv[1], dtype=np.int64)
base = a[0][0]
print(" chunk  split_free   split_st  mma_seen  mma_commit   (cycles rel. to first TMA issue)")
for i in range(16, 40):
    print(f"{i//8}.{i%8}  " + " ".join(f"{(a[k][i]-base) if a[k][i] else -1:>10d}" for k in (8, 9, 10, 11)))
