import sys, torch, time
sys.path.insert(0, '.')
import synth, paper_2507_23207_b200 as krp
cfg = synth.config("c5")
x = torch.from_numpy(synth.tensor(cfg, 0)).cuda()
om = [torch.from_numpy(o).cuda() for o in synth.omegas(cfg.dims, cfg.R, 0)]
ws = torch.empty(krp.krp_workspace_bytes(krp.OP_RHOSVD, cfg.dims, cfg.R, cfg.ranks), dtype=torch.uint8, device="cuda")
run = lambda: krp.krp_rhosvd(x, cfg.dims, cfg.ranks, om, ws=ws)
for _ in range(2): run()
torch.cuda.synchronize()
evs = []
t0 = time.time()
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); run(); b.record(); evs.append((a, b))
torch.cuda.synchronize()
print("host s per call %.3f ms" % ((time.time() - t0) * 100))
print("per call ms:", " ".join("%.2f" % a.elapsed_time(b) for a, b in evs))
time.sleep(2)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); run(); b.record(); torch.cuda.synchronize(); print("after 2 s idle: %.2f ms" % a.elapsed_time(b))
