"""The sharded (NCCL) entry points on one GPU with a one-rank process group: the packing of partial
sketches and slab rows, the NCCL all-reduce call and the unpacking run for real.

With one rank the all-reduce is the identity, so:
  * the whole tensor as one "slab" must reproduce krp_sketch_all_modes / krp_rhosvd exactly;
  * a partial slab [k0, k1) of a longer last mode must give the partial sketches of that slab
    (Y_1..Y_{d-1} of the slab tensor) and Y_d rows k0..k1 of the global sketch, zeros elsewhere.
Multi-rank sums are covered on CPU by tests/test_dist_gloo.py (world size 2)."""
import os
import socket

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


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
    for a, b in zip(got, ref):
        assert torch.equal(a, b)


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
    # the same slab sketched as a standalone tensor with the slab's rows of Ω_3
    om_slab = [om[0], om[1], _dev(om_np[2][k0:k1])]
    ref = krp.krp_sketch_all_modes(_dev(slab), dims_local, om_slab)
    torch.cuda.synchronize()
    assert torch.equal(got[0], ref[0]) and torch.equal(got[1], ref[1])
    y3 = got[2].cpu()
    assert torch.equal(y3[k0:k1], ref[2].cpu())
    assert float(y3[:k0].abs().max()) == 0.0 and float(y3[k1:].abs().max()) == 0.0


def test_dist_rhosvd_whole_tensor_equals_single_gpu(env):
    krp, comm = env
    cfg = synth.config("c2").scaled((96, 80, 64))
    x = _dev(synth.tensor(cfg, 3))
    om = [_dev(o) for o in synth.omegas(cfg.dims, cfg.R, 3)]
    _, _, e1 = krp.krp_rhosvd(x, cfg.dims, cfg.ranks, om, with_error=True)
    _, _, e2 = krp.krp_rhosvd_dist(x, cfg.dims, cfg.dims[-1], 0, cfg.ranks, om, comm, with_error=True)
    assert abs(e1 - e2) <= 1e-7 * max(1.0, abs(e1)), (e1, e2)
