"""Where does the GPU's extra c5 Tucker error come from (dev tool)?  e(Q_gpu, G_gpu) vs e(Q_gpu, G64) where
G64 = X x_n Q_gpu,n^T in fp64 (the optimal core for the GPU's subspaces), vs the oracle's own error."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import synth, oracle
from oracle import krp_oracle as _ko
import paper_2507_23207_b200 as krp
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
cfg = synth.config(name)
x = synth.tensor(cfg, 0)
om = synth.omegas(cfg.dims, cfg.R, 0)
Q, core, err = krp.krp_rhosvd(torch.from_numpy(x).cuda(), cfg.dims, cfg.ranks, [torch.from_numpy(o).cuda() for o in om],
                              with_error=True)
X = oracle.as_tensor(x, cfg.dims)
qs = [q.double().cpu().numpy() for q in Q]
g = core.double().cpu().numpy().reshape(cfg.ranks, order="F")
ch = max(1, cfg.dims[-1] // 16)
e_gg = oracle.tucker_error(X, g, qs, chunk=ch)
g64 = _ko._core_slabwise(X, qs, ch)
e_g64 = oracle.tucker_error(X, g64, qs, chunk=ch)
print(f"{name}: gpu-reported {err:.6e}  e(Q_gpu, G_gpu) {e_gg:.6e}  e(Q_gpu, G64) {e_g64:.6e}  "
      f"core rel diff {np.linalg.norm(g - g64) / np.linalg.norm(g64):.3e}", flush=True)
qo, go, eo, _ = oracle.rhosvd(X, om, cfg.ranks, chunk=ch)
print(f"oracle {eo:.6e}; subspace gaps: " + ", ".join(
    f"{np.linalg.norm(qo[n] @ (qo[n].T @ qs[n]) - qs[n]):.3e}" for n in range(cfg.d)), flush=True)
