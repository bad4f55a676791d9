"""Time the sketch on a config (dev tool): per-kernel event timing via the library profiler."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import synth, oracle
import paper_2507_23207_b200 as krp
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
check = len(sys.argv) > 3
if name.startswith("dims:"):  # dims:64,64,64,64,8:20 -> a random tensor of that shape, R = 20
    _, ds, rs = name.split(":")
    class _C: pass
    cfg = _C(); cfg.dims = tuple(int(v) for v in ds.split(",")); cfg.R = int(rs); cfg.N = int(np.prod(cfg.dims))
else:
    cfg = synth.config(name)
dims = cfg.dims
xn = synth.random_tensor(dims, 1)
x = torch.from_numpy(xn).cuda()
omn = synth.omegas(dims, cfg.R, 2)
om = [torch.from_numpy(o).cuda() for o in omn]
ws = torch.empty(krp.krp_workspace_bytes(krp.OP_SKETCH_ALL, dims, cfg.R), dtype=torch.uint8, device='cuda')
Y = [torch.empty((n, cfg.R), device='cuda') for n in dims]
for _ in range(3 if len(sys.argv) < 5 else 0):
    krp.krp_sketch_all_modes(x, dims, om, Y=Y, ws=ws)
torch.cuda.synchronize()
krp.krp_profile_reset(); krp.krp_profile_enable(True)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    krp.krp_sketch_all_modes(x, dims, om, Y=Y, ws=ws)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
kms, kn, kb, kf = krp.krp_profile_read()
print(f"{name}: step {ms*1e3:.1f} us, main kernel {kms/kn*1e3:.1f} us -> {kb/kn/(kms/kn*1e-3)/1e9:.0f} GB/s, "
      f"{4*cfg.N*cfg.R/(ms*1e-3)/1e12:.1f} alg TFLOP/s (step)")
if check:
    rows = [0, 1, dims[0] // 2, dims[0] - 1]
    for n in range(len(dims)):
        rr = [0, 7, dims[n] - 1]
        ref = oracle.sketch_mode_rows(xn, dims, omn, n, rr)
        got = Y[n].double().cpu().numpy()[rr]
        print("mode", n, "sampled rel err %.2e" % (np.linalg.norm(got - ref) / np.linalg.norm(ref)))
