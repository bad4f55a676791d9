"""Per-rank work of the slab-sharded sketch at N = 1, 2, 4, 8, measured on ONE GPU (dev tool).

Runs krp_sketch_all_modes_dist on rank 0's slab of an N-way split with a one-rank NCCL communicator
(the all-reduce is then a local pass over the packed buffer), so the numbers are the per-rank compute +
packing time of the N-GPU step without the multi-rank collective.  usage: slab_time.py <config> [steps] [worlds, e.g. 1,8]
"""
import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2507_23207_b200 as krp  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    worlds = [int(w) for w in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 2, 4, 8]
    cfg = synth.config(name)
    torch.cuda.set_device(0)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    comm = krp.Comm()
    Id = cfg.dims[-1]
    om = [torch.from_numpy(o).cuda() for o in synth.omegas(cfg.dims, cfg.R, 0)]
    Y = [torch.empty((n, cfg.R), dtype=torch.float32, device="cuda") for n in cfg.dims]
    base = None
    for world in worlds:
        k0, kn = krp.krp_slab_range(Id, world, 0)
        dims_local = list(cfg.dims[:-1]) + [kn]
        X = torch.from_numpy(synth.tensor_slab(cfg, 0, k0, k0 + kn)).cuda()
        ws = torch.empty(krp.krp_workspace_bytes_dist(krp.OP_SKETCH_ALL, dims_local, Id, cfg.R), dtype=torch.uint8,
                         device="cuda")

        def step():
            krp.krp_sketch_all_modes_dist(X, dims_local, Id, k0, om, comm, Y=Y, ws=ws)

        for _ in range(5):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        if base is None:
            base = ms
        print(f"{name} N={world}: slab {kn}/{Id}, per-rank step {ms * 1e3:8.1f} us, "
              f"ideal {base / world * 1e3:8.1f} us, compute-side efficiency {base / world / ms:5.2f}")
        del X, ws
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
