"""One c3 STHOSVD (dev tool) for an ncu launch list: python tools/sthosvd_launches.py [cfg]"""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
import synth
import paper_2507_23207_b200 as krp
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = synth.config(name)
x = torch.randn(cfg.N, device="cuda")
oms = synth.sthosvd_omegas(cfg.dims, cfg.R, 0)
dom = [[None if o is None else torch.from_numpy(o).cuda() for o in row] for row in oms]
for _ in range(2):
    krp.krp_sthosvd(x, cfg.dims, cfg.ranks, dom)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
krp.krp_sthosvd(x, cfg.dims, cfg.ranks, dom)
e1.record()
torch.cuda.synchronize()
print(f"{name} sthosvd {e0.elapsed_time(e1):.3f} ms")
