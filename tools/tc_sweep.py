"""Sketch kernel time vs last-mode length (dev tool): fits kernel_us = a * tiles_per_CTA + b."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import synth
import paper_2507_23207_b200 as krp
I, R = int(sys.argv[1]) if len(sys.argv) > 1 else 512, int(sys.argv[2]) if len(sys.argv) > 2 else 40
pts = []
for S in (8, 16, 32, 64, 128, 256, 512):
    dims = (I, I, S)
    x = torch.from_numpy(synth.random_tensor(dims, 1)).cuda()
    om = [torch.from_numpy(o).cuda() for o in synth.omegas(dims, R, 2)]
    ws = torch.empty(krp.krp_workspace_bytes(krp.OP_SKETCH_ALL, dims, R), dtype=torch.uint8, device='cuda')
    Y = [torch.empty((n, R), device='cuda') for n in dims]
    for _ in range(3):
        krp.krp_sketch_all_modes(x, dims, om, Y=Y, ws=ws)
    torch.cuda.synchronize()
    krp.krp_profile_reset(); krp.krp_profile_enable(True)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        krp.krp_sketch_all_modes(x, dims, om, Y=Y, ws=ws)
    e1.record(); torch.cuda.synchronize()
    krp.krp_profile_enable(False)
    kms, kn, kb, kf = krp.krp_profile_read()
    tiles = (I // 128) ** 2 * S / 148.0
    step = e0.elapsed_time(e1) / 20 * 1e3
    pts.append((tiles, kms / kn * 1e3))
    print(f"dims {dims}: tiles/CTA {tiles:6.2f}  kernel {kms / kn * 1e3:7.1f} us  step {step:7.1f} us")
t = np.array(pts)
a, b = np.polyfit(t[:, 0], t[:, 1], 1)
print(f"fit: kernel_us = {a:.2f} * tiles_per_CTA + {b:.1f}")
