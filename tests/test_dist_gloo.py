"""World-size-2 CPU tests (gloo) of the sharded path's host logic.

The GPU kernels cannot run here, so every rank computes its slab's partial sketches with the fp64 oracle
(test infrastructure) and places them with the LIBRARY's host geometry (krp_slab_range, krp_pack_layout —
the same functions krp_sketch_all_modes_dist uses); one all-reduce(sum) over gloo must then reproduce the
unsharded oracle sketch exactly (to fp64 rounding): partial Y_1..Y_{d-1} summed, Y_d slab rows gathered."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dims, R, seed, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2507_23207_b200 as krp
        from paper_2507_23207_b200 import build
        build.build()
        d = len(dims)
        Id = dims[-1]
        b, n = krp.krp_slab_range(Id, world, rank)
        x = synth.random_tensor(dims, seed, d)
        om = synth.omegas(dims, R, seed)
        inner = int(np.prod(dims[:-1]))
        slab = x[b * inner:(b + n) * inner]
        dims_local = list(dims[:-1]) + [n]
        oms = list(om[:-1]) + [om[-1][b:b + n]]
        ys = oracle.sketch_all_modes(oracle.as_tensor(slab, dims_local), oms) if n > 0 else None
        offs, soff = krp.krp_pack_layout(dims_local, Id, b, R)
        buf = torch.zeros(offs[-1], dtype=torch.float64)
        if ys is not None:
            for k in range(d - 1):
                buf[offs[k]:offs[k + 1]] = torch.from_numpy(ys[k].reshape(-1))
            buf[soff:soff + n * R] = torch.from_numpy(ys[d - 1].reshape(-1))
        dist.all_reduce(buf, op=dist.ReduceOp.SUM)
        ref = oracle.sketch_all_modes(oracle.as_tensor(x, dims), om)
        err = 0.0
        for k in range(d):
            got = buf[offs[k]:offs[k + 1]].numpy().reshape(-1, R)
            err = max(err, float(np.abs(got - ref[k]).max() / np.abs(ref[k]).max()))
        q.put((rank, b, n, offs, err))
        dist.destroy_process_group()
    except Exception as e:  # surface the failure in the parent
        q.put((rank, "error", repr(e)))


@pytest.mark.parametrize("dims,R", [((6, 5, 8), 3), ((4, 3, 5, 7), 4), ((7, 3, 2, 2, 3), 2)])
def test_two_rank_slab_sharded_sketch_matches_unsharded(dims, R):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, R, 3, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    out.sort(key=lambda t: t[0])
    for o in out:
        assert o[1] != "error", o
    # the slabs tile [0, I_d) contiguously (ragged split when world does not divide I_d)
    assert out[0][1] == 0 and out[0][1] + out[0][2] == out[1][1] and out[1][1] + out[1][2] == dims[-1]
    assert out[0][3] == out[1][3]  # both ranks agree on the packed layout
    for o in out:
        assert o[4] < 1e-12, o


def test_slab_range_and_pack_layout_host_only():
    import paper_2507_23207_b200 as krp
    from paper_2507_23207_b200 import build
    build.build()
    for Id in (1, 7, 64, 512):
        for G in (1, 2, 3, 8):
            if G > Id:  # every rank must own a non-empty slab: all ranks fail together, before any collective
                with pytest.raises(krp.KrpError):
                    krp.krp_slab_range(Id, G, 0)
                continue
            spans = [krp.krp_slab_range(Id, G, g) for g in range(G)]
            assert spans[0][0] == 0 and sum(n for _, n in spans) == Id
            for (b0, n0), (b1, _) in zip(spans, spans[1:]):
                assert b0 + n0 == b1
            assert max(n for _, n in spans) - min(n for _, n in spans) <= 1
    offs, soff = krp.krp_pack_layout([5, 6, 3], 10, 4, 2)
    assert offs == [0, 10, 22, 42] and soff == 22 + 4 * 2
    with pytest.raises(krp.KrpError):
        krp.krp_slab_range(8, 2, 2)
    with pytest.raises(krp.KrpError):
        krp.krp_pack_layout([5, 6, 3], 10, 8, 2)  # slab [8, 11) exceeds I_d = 10
