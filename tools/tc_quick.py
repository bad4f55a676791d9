"""Quick TC-engine check on a few shapes (dev tool)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import synth, oracle
import paper_2507_23207_b200 as krp
krp.krp_set_engine(1)
shapes = [((128,128,4),16), ((256,256,8),40), ((512,512,16),40), ((200,136,5),10), ((128,128,40),64), ((16,16,16,16,16),20)]
for dims, R in shapes:
    x = synth.random_tensor(dims, 1, len(dims)); om = synth.omegas(dims, R, 2)
    ref = oracle.sketch_all_modes(oracle.as_tensor(x, dims), om)
    try:
        Y = krp.krp_sketch_all_modes(torch.from_numpy(x).cuda(), dims, [torch.from_numpy(o).cuda() for o in om])
        torch.cuda.synchronize()
        errs = [float(np.linalg.norm(Y[n].double().cpu().numpy()-ref[n])/np.linalg.norm(ref[n])) for n in range(len(dims))]
        print(dims, R, ["%.2e" % e for e in errs], flush=True)
    except krp.KrpError as e:
        print(dims, R, "ERR", e, flush=True)
