"""The sharded (NCCL) entry points on one GPU with a one-rank process group: the packing of partial
sketches and slab rows, the NCCL all-reduce call and the unpacking run for real.

With one rank the all-reduce is the identity, so:
  * the whole tensor as one "slab" must match the fp64 oracle (and krp_sketch_all_modes bit for bit);
  * a partial slab [k0, k1) of a longer last mode must give the oracle's partial sketches of that slab
    (Y_1..Y_{d-1} of the slab tensor) and its Y_d rows k0..k1, zeros elsewhere;
  * krp_rhosvd_dist on the whole tensor matches the oracle's rHOSVD error.
Multi-rank sums are covered on CPU by tests/test_dist_gloo.py (world size 2) and, when the box has two
GPUs, by test_two_rank_nccl_sketch_matches_oracle (torch.multiprocessing, NCCL)."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
Y_TOL = 1e-5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist
    import paper_2507_23207_b200 as krp
    from paper_2507_23207_b200 import build
    build.build()
    torch.cuda.set_device(0)
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    comm = krp.Comm()
    yield krp, comm
    comm.close()
    dist.destroy_process_group()


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


@pytest.mark.parametrize("dims,R", [((64, 48, 40), 10), ((32, 16, 24, 20), 8)])
def test_dist_whole_tensor_equals_single_gpu(env, dims, R):
    krp, comm = env
    x = synth.random_tensor(dims, 21, len(dims))
    om = [_dev(o) for o in synth.omegas(dims, R, 22)]
    X = _dev(x)
    ref = krp.krp_sketch_all_modes(X, dims, om)
    got = krp.krp_sketch_all_modes_dist(X, dims, dims[-1], 0, om, comm)
    torch.cuda.synchronize()
    oref = oracle.sketch_all_modes(oracle.as_tensor(x, dims), synth.omegas(dims, R, 22))
    for a, b, o in zip(got, ref, oref):
        assert torch.equal(a, b)
        assert np.linalg.norm(a.double().cpu().numpy() - o) / np.linalg.norm(o) <= Y_TOL


def test_dist_partial_slab_packing(env):
    krp, comm = env
    dims, R = (64, 40, 30), 12
    k0, k1 = 7, 19
    x = synth.random_tensor(dims, 23, 3)
    om_np = synth.omegas(dims, R, 24)
    inner = dims[0] * dims[1]
    slab = x[k0 * inner:k1 * inner]
    dims_local = (dims[0], dims[1], k1 - k0)
    om = [_dev(o) for o in om_np]
    got = krp.krp_sketch_all_modes_dist(_dev(slab), dims_local, dims[-1], k0, om, comm)
    # the oracle's sketch of the slab as a standalone tensor with the slab's rows of Ω_3
    oref = oracle.sketch_all_modes(oracle.as_tensor(slab, dims_local), [om_np[0], om_np[1], om_np[2][k0:k1]])
    torch.cuda.synchronize()
    for n in range(2):
        assert np.linalg.norm(got[n].double().cpu().numpy() - oref[n]) / np.linalg.norm(oref[n]) <= Y_TOL
    y3 = got[2].double().cpu().numpy()
    assert np.linalg.norm(y3[k0:k1] - oref[2]) / np.linalg.norm(oref[2]) <= Y_TOL
    assert np.abs(y3[:k0]).max() == 0.0 and np.abs(y3[k1:]).max() == 0.0


def test_dist_rhosvd_whole_tensor_equals_single_gpu(env):
    krp, comm = env
    cfg = synth.config("c2").scaled((96, 80, 64))
    x = _dev(synth.tensor(cfg, 3))
    om = [_dev(o) for o in synth.omegas(cfg.dims, cfg.R, 3)]
    _, _, e1 = krp.krp_rhosvd(x, cfg.dims, cfg.ranks, om, with_error=True)
    _, _, e2 = krp.krp_rhosvd_dist(x, cfg.dims, cfg.dims[-1], 0, cfg.ranks, om, comm, with_error=True)
    assert abs(e1 - e2) <= 1e-7 * max(1.0, abs(e1)), (e1, e2)
    xn = synth.tensor(cfg, 3)
    _, _, eref, _ = oracle.rhosvd(oracle.as_tensor(xn, cfg.dims), synth.omegas(cfg.dims, cfg.R, 3), cfg.ranks)
    assert abs(e2 - eref) <= 1e-4, (e2, eref)


def test_dist_sthosvd_whole_tensor_matches_oracle(env):
    """krp_sthosvd_dist with the whole tensor as one slab: the single-GPU decomposition and the oracle's error."""
    krp, comm = env
    cfg = synth.config("c3").scaled((40, 36, 32, 32))
    x = synth.tensor(cfg, 5)
    oms = synth.sthosvd_omegas(cfg.dims, cfg.R, 5)
    dom = [[None if o is None else _dev(o) for o in row] for row in oms]
    _, _, e1 = krp.krp_sthosvd(_dev(x), cfg.dims, cfg.ranks, dom, with_error=True)
    Q, core, e2 = krp.krp_sthosvd_dist(_dev(x), cfg.dims, cfg.dims[-1], 0, cfg.ranks, dom, comm, with_error=True)
    assert abs(e1 - e2) <= 1e-7 * max(1.0, abs(e1)), (e1, e2)
    _, _, eref, _ = oracle.sthosvd(oracle.as_tensor(x, cfg.dims), oms, cfg.ranks)
    assert abs(e2 - eref) <= 1e-4, (e2, eref)
    for q, r in zip(Q, cfg.ranks):
        qq = q.double().cpu().numpy()
        assert np.abs(qq.T @ qq - np.eye(r)).max() <= 1e-6


def _nccl_worker(rank, world, port, q):
    """One rank of a 2-GPU run: sketch the rank's slab with the NCCL combine, compare with the oracle."""
    try:
        import os
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
        import paper_2507_23207_b200 as krp
        dims, R = (96, 80, 37), 12  # ragged split of the last mode
        x = synth.random_tensor(dims, 31, 3)
        om_np = synth.omegas(dims, R, 32)
        b, n = krp.krp_slab_range(dims[-1], world, rank)
        inner = dims[0] * dims[1]
        slab = x[b * inner:(b + n) * inner]
        comm = krp.Comm()
        Y = krp.krp_sketch_all_modes_dist(_dev(slab), (dims[0], dims[1], n), dims[-1], b,
                                          [_dev(o) for o in om_np], comm)
        torch.cuda.synchronize()
        ref = oracle.sketch_all_modes(oracle.as_tensor(x, dims), om_np)
        err = max(float(np.linalg.norm(y.double().cpu().numpy() - r) / np.linalg.norm(r)) for y, r in zip(Y, ref))
        # sharded STHOSVD (Alg. 8) of a Tucker tensor vs the oracle's error
        cfg = synth.config("c3").scaled((40, 36, 32, 32))
        xt = synth.tensor(cfg, 6)
        oms = synth.sthosvd_omegas(cfg.dims, cfg.R, 6)
        b2, n2 = krp.krp_slab_range(cfg.dims[-1], world, rank)
        inn = int(np.prod(cfg.dims[:-1]))
        dom = [[None if o is None else _dev(o) for o in row] for row in oms]
        _, _, es = krp.krp_sthosvd_dist(_dev(xt[b2 * inn:(b2 + n2) * inn]), list(cfg.dims[:-1]) + [n2],
                                        cfg.dims[-1], b2, cfg.ranks, dom, comm, with_error=True)
        _, _, eref, _ = oracle.sthosvd(oracle.as_tensor(xt, cfg.dims), oms, cfg.ranks)
        if abs(es - eref) > 1e-4:
            err = max(err, 1.0)
        comm.close()
        dist.destroy_process_group()
        q.put((rank, err))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, repr(e)))


def test_two_rank_nccl_sketch_matches_oracle():
    """The sharded sketch over NCCL on two GPUs (runs only where the box has two)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for rank, err in out:
        assert isinstance(err, float) and err <= Y_TOL, (rank, err)
