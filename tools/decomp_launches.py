"""One timed rHOSVD / STHOSVD call (dev tool, for an ncu launch list):
python tools/decomp_launches.py {rhosvd|sthosvd} [cfg]"""
import sys
import torch
sys.path.insert(0, '.')
import synth
import paper_2507_23207_b200 as krp
alg = sys.argv[1]
name = sys.argv[2] if len(sys.argv) > 2 else ("c5" if alg == "rhosvd" else "c3")
cfg = synth.config(name)
x = torch.from_numpy(synth.tensor(cfg, 0)).cuda()  # the config's own data (spectra drive the eigensolver)
if alg == "rhosvd":
    om = [torch.from_numpy(o).cuda() for o in synth.omegas(cfg.dims, cfg.R, 0)]
    ws = torch.empty(krp.krp_workspace_bytes(krp.OP_RHOSVD, cfg.dims, cfg.R, cfg.ranks), dtype=torch.uint8, device="cuda")
    run = lambda: krp.krp_rhosvd(x, cfg.dims, cfg.ranks, om, ws=ws)
else:
    oms = synth.sthosvd_omegas(cfg.dims, cfg.R, 0)
    dom = [[None if o is None else torch.from_numpy(o).cuda() for o in row] for row in oms]
    ws = torch.empty(krp.krp_workspace_bytes(krp.OP_STHOSVD, cfg.dims, cfg.R, cfg.ranks), dtype=torch.uint8, device="cuda")
    run = lambda: krp.krp_sthosvd(x, cfg.dims, cfg.ranks, dom, ws=ws)
for _ in range(2):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run()
e1.record()
torch.cuda.synchronize()
print(f"{name} {alg} {e0.elapsed_time(e1):.3f} ms")
