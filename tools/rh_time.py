"""Time krp_rhosvd / krp_sthosvd on a config (dev tool)."""
import sys, time, torch
sys.path.insert(0, '.')
import synth
import paper_2507_23207_b200 as krp
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = synth.config(name)
x = torch.from_numpy(synth.random_tensor(cfg.dims, 1)).cuda()
if cfg.workload == "sthosvd":
    oms = [[None if o is None else torch.from_numpy(o).cuda() for o in row] for row in synth.sthosvd_omegas(cfg.dims, cfg.R, 2)]
    fn = lambda: krp.krp_sthosvd(x, cfg.dims, cfg.ranks, oms)
else:
    om = [torch.from_numpy(o).cuda() for o in synth.omegas(cfg.dims, cfg.R, 2)]
    fn = lambda: krp.krp_rhosvd(x, cfg.dims, cfg.ranks, om)
for _ in range(2): fn()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(steps): fn()
torch.cuda.synchronize()
print(f"{name} {cfg.workload}: {(time.perf_counter() - t) / steps * 1e3:.2f} ms per call")
