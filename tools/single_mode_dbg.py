import sys, numpy as np, torch
sys.path.insert(0, '.')
import synth, oracle
import paper_2507_23207_b200 as krp
krp.krp_set_engine(1)
dims, R = (128, 128, 128), 30
x = synth.random_tensor(dims, 3, 3); om = synth.omegas(dims, R, 4)
X = oracle.as_tensor(x, dims)
for n in range(3):
    omn = [None if k == n else torch.from_numpy(o).cuda() for k, o in enumerate(om)]
    try:
        Y = krp.krp_sketch_mode(torch.from_numpy(x).cuda(), dims, n, omn)
        torch.cuda.synchronize()
        ref = oracle.sketch_mode(X, om, n)
        print(n, "err %.2e" % (np.linalg.norm(Y.double().cpu().numpy() - ref) / np.linalg.norm(ref)), flush=True)
    except Exception as e:
        print(n, "FAILED", repr(e)[:300], flush=True)
        break
