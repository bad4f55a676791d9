"""NEXT-1: the paper's Cauchy-tensor experiment (Fig. 2 / Fig. 3 setup) on one B200.

4-way Cauchy tensor, n = 250, a = 2 (15.6 GB fp32, generated on the device), target rank r swept with no
oversampling (R = r).  For each r: RHOSVD-KRP-MEMO (krp_rhosvd) and RSTHOSVD-KRP (krp_sthosvd)
relative errors (the library's own error pass) and device times (CUDA events), plus the memoized all-mode
sketch time.  Context at a reduced n (the fp64 oracle, host): HOSVD, STHOSVD and the oracle's randomized
errors at the same ranks.  Writes profiles/<tag>_cauchy_sweep.json and prints one line per rank.

  python tools/cauchy_sweep.py [tag] [n] [n_small]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2507_23207_b200 as krp  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 250
n_small = int(sys.argv[3]) if len(sys.argv) > 3 else 40
ranks_sweep = [5, 10, 15, 20, 25, 30]
dims = (n,) * 4
dev = torch.device("cuda", 0)
t0 = time.time()
X = synth.cauchy_device(dims, 2.0, device=dev)
torch.cuda.synchronize()
gen_s = time.time() - t0


def ev_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3, out


rows = []
for r in ranks_sweep:
    om = [torch.from_numpy(o).to(dev) for o in synth.omegas(dims, r, 0)]
    oms = [[None if o is None else torch.from_numpy(o).to(dev) for o in row] for row in synth.sthosvd_omegas(dims, r, 0)]
    rk = (r,) * 4
    t_sk, _ = ev_time(lambda: krp.krp_sketch_all_modes(X, dims, om))
    t_rh, _ = ev_time(lambda: krp.krp_rhosvd(X, dims, rk, om))
    t_st, _ = ev_time(lambda: krp.krp_sthosvd(X, dims, rk, oms))
    e_rh = krp.krp_rhosvd(X, dims, rk, om, with_error=True)[2]
    e_st = krp.krp_sthosvd(X, dims, rk, oms, with_error=True)[2]
    row = {"r": r, "R": r, "rhosvd_memo_err": e_rh, "sthosvd_krp_err": e_st, "sketch_all_s": t_sk,
           "rhosvd_memo_s": t_rh, "sthosvd_krp_s": t_st,
           "sketch_tflops": 4.0 * float(np.prod(dims)) * r / t_sk / 1e12}
    rows.append(row)
    print(json.dumps(row), flush=True)
    del om, oms
    torch.cuda.empty_cache()
del X
torch.cuda.empty_cache()

# context at a reduced n: the fp64 oracle's deterministic and randomized errors at the same ranks
small = []
try:
    import oracle
    cs = synth.config("cauchy").scaled((n_small,) * 4)
    xs = oracle.as_tensor(synth.tensor(cs, 0), cs.dims)
    xsd = torch.from_numpy(synth.tensor(cs, 0)).to(dev)
    for r in ranks_sweep:
        if r > n_small // 2:
            continue
        rk = (r,) * 4
        om = synth.omegas(cs.dims, r, 0)
        oms = synth.sthosvd_omegas(cs.dims, r, 0)
        ent = {"n": n_small, "r": r, "hosvd_err": oracle.hosvd(xs, rk)[2],
               "sthosvd_det_err": oracle.sthosvd_deterministic(xs, rk)[2],
               "oracle_rhosvd_memo_err": oracle.rhosvd(xs, om, rk)[2],
               "oracle_sthosvd_krp_err": oracle.sthosvd(xs, oms, rk)[2],
               "gpu_rhosvd_memo_err": krp.krp_rhosvd(xsd, cs.dims, rk, [torch.from_numpy(o).to(dev) for o in om],
                                                     with_error=True)[2],
               "gpu_sthosvd_krp_err": krp.krp_sthosvd(xsd, cs.dims, rk, [[None if o is None else torch.from_numpy(o).to(dev)
                                                                         for o in row] for row in oms],
                                                      with_error=True)[2]}
        small.append(ent)
        print(json.dumps(ent), flush=True)
except Exception as e:  # the context leg is optional
    print("small-n context skipped:", repr(e))

out = {"workload": f"Cauchy tensor n={n}, a=2, 4-way (P:712-725), R = r (no oversampling), device-generated "
                   f"({gen_s:.1f} s)", "gpu": torch.cuda.get_device_name(0), "sweep": rows, "small_n_context": small}
os.makedirs("profiles", exist_ok=True)
with open(f"profiles/{tag}_cauchy_sweep.json", "w") as f:
    json.dump(out, f, indent=1)
print("wrote", f"profiles/{tag}_cauchy_sweep.json")
