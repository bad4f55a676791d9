"""Quick sketch check on a few shapes (dev tool): relative error per mode vs the fp64 oracle."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import synth, oracle
import paper_2507_23207_b200 as krp
shapes = [((128,128,4),16), ((256,256,8),40), ((512,512,16),40), ((200,136,5),10), ((128,128,40),64),
          ((16,16,16,16,16),20), ((64,64,64),10), ((5,7,9),4), ((300,260),33), ((128,96,20),100)]
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
