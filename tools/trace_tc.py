"""Print the KRP_DEV_TRACE timeline of CTAs 0/1 (dev tool).  usage: python tools/trace_tc.py trace.txt [ntiles]"""
import sys
import numpy as np
rows = [list(map(int, l.split())) for l in open(sys.argv[1])]
a = np.array(rows, dtype=np.int64).reshape(2, 16, 64)
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 12
t0 = min(v for v in a.reshape(-1) if v > 0)
names = {0: "tma_wait_empty", 1: "tma_issue", 2: "mma_start", 3: "mma_end", 4: "split_wait_full", 5: "split_full",
         6: "split0_done", 7: "split4_done", 8: "epi_wait", 9: "epi_acc_full", 10: "epi_done", 11: "b_ready",
         12: "epi_ld1", 13: "epi_Tbar"}
for c in range(2):
    print(f"--- CTA {c} (us from first event)")
    print("tile " + " ".join(f"{names[k][:13]:>13s}" for k in sorted(names)))
    for t in range(nt):
        print(f"{t:4d} " + " ".join(f"{(a[c, k, t] - t0) / 1e3:13.2f}" if a[c, k, t] > 0 else f"{'-':>13s}"
                                    for k in sorted(names)))
    for k in (1, 3, 6, 10):
        v = a[c, k, :]
        v = v[v > 0]
        if len(v) > 4:
            print(f"  {names[k]} mean period {np.mean(np.diff(v)) / 1e3:.3f} us over {len(v)} tiles")

secs = ["oms/loop-top->wait", "acc_full wait", "tmem ld+wait (batch)", "math", "arrive->Tbar", "Tbar wait", "Tsum+STG", "loop/segment"]
for c in range(2):
    print(f"--- CTA {c} epilogue section cycles per tile (sum over the kernel / 64*?)")
    for w in range(8):
        row = a[c, 14 + (w >> 2), (w & 3) * 8:(w & 3) * 8 + 8]
        tot = row.sum()
        print(f"  warp {w}: " + "  ".join(f"{secs[i][:10]}={row[i]:.3g}" for i in range(8)) + f"  total={tot:.3g}")
