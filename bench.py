#!/usr/bin/env python
"""bench.py — all-mode KRP sketch throughput (and rHOSVD time) on B200, BASELINE.json's metric.

Default (N=1): BASELINE configs[1] = c2, a 512^3 fp32 Tucker(30^3, decay 0.8) + 1e-3 noise tensor,
R = 40, inputs resident in HBM (512 MiB > 126 MB L2, so no L2 flush is needed between steps).

One timed step of the headline = one krp_sketch_all_modes call (memoized all-mode sketch, SURVEY
§8(a) rows a1-a6, including the NCCL combine at N>1).  The same run also times K full rHOSVD steps
(rows a1-a9: sketch, CholeskyQR, core, truncation) -> "rhosvd_s".
value = 4*N*R*K / t  (algorithmic TFLOP/s), t = max over ranks of CUDA-event time.

  python bench.py [--gpus N --steps K --warmup W] [--config c5]
  python bench.py --impl reference ...   # the fp64 oracle on host cores (bounded sample per step)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "all-mode KRP sketch TFLOP/s & % roofline (3xTF32 vs HBM), rHOSVD s, 1/2/4/8 GPU"


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), float(mp["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"  # B200_PROFILING.md fallback figures


def _workload(cfg, world):
    return {
        "workload": f"{cfg.name}: {'x'.join(map(str, cfg.dims))} fp32 "
                    + (f"Tucker core {'x'.join(map(str, cfg.core))}" + (f" decay {cfg.decay}" if cfg.decay else "")
                       if cfg.kind == "tucker" else "smooth 1/(1+i/I1+j/I2+k/I3)")
                    + f" + {cfg.eta:g} rel. noise, R={cfg.R}, memoized all-mode KRP sketch (+ rHOSVD to ranks "
                    + f"{'x'.join(map(str, cfg.ranks))})",
        "dims": list(cfg.dims),
        "R": cfg.R,
        "ranks": list(cfg.ranks),
        "sharding": f"slabs along mode {cfg.d} over {world} GPU(s)",
        "l2": "inputs larger than L2 (no flush needed)" if 4 * cfg.N > 126e6 * 1.5 else "L2 flushed between steps",
    }


# ------------------------------------------------------------------ clocks (nvidia-smi during the timed region)
class ClockSampler:
    """SM clock + throttle reasons polled through NVML (~1 ms) during the timed region; falls back to
    `nvidia-smi -lms 200` when NVML is unavailable."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self.stop_ev = threading.Event()
        self.th = None
        self.smax = None

    def _poll(self):
        import pynvml
        h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
        self.smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while not self.stop_ev.is_set():
            try:
                clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((clk, rs))
            except Exception:
                pass
            time.sleep(0.001)

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.th = threading.Thread(target=self._poll, daemon=True)
            self.th.start()
            t0 = time.time()
            while not self.samples and time.time() - t0 < 1.0:  # the timed region starts once sampling runs
                time.sleep(0.001)
        except Exception:
            self.th = None

    def stop(self):
        if self.th is None:
            return None
        self.stop_ev.set()
        self.th.join(timeout=2)
        if not self.samples:
            return None
        reasons = sorted({nm for _, rs in self.samples for nm, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(c for c, _ in self.samples), "sm_max_mhz": self.smax,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml"}


# ------------------------------------------------------------------ CPU oracle baseline
def _oracle_sample(cfg, seed, slabs, om):
    import oracle
    x = synth.tensor_slab(cfg, seed, 0, slabs)
    dims = list(cfg.dims[:-1]) + [slabs]
    oms = list(om[:-1]) + [om[-1][:slabs]]
    X = oracle.as_tensor(x, dims)
    t0 = time.perf_counter()
    oracle.sketch_all_modes(X, oms)
    t = time.perf_counter() - t0
    flops = oracle.sketch_flops(dims, cfg.R)
    return t, flops


def _cores():
    try:
        from threadpoolctl import threadpool_info
        nt = max((int(p.get("num_threads", 1)) for p in threadpool_info()), default=1)
    except Exception:
        nt = os.cpu_count() or 1
    return nt


def _calibrate_slabs(cfg, seed, om, target_s):
    """Number of last-mode slabs whose oracle sketch takes about target_s (doubling calibration)."""
    slabs, t = 1, 0.0
    while slabs < cfg.dims[-1]:
        t, _ = _oracle_sample(cfg, seed, slabs, om)
        if t >= 0.25 * target_s:
            break
        slabs = min(cfg.dims[-1], slabs * 2)
    if t > 0:
        slabs = int(max(1, min(cfg.dims[-1], slabs * target_s / t)))
    return slabs


def cpu_baseline(cfg, seed, om, target_s=12.0):
    """The oracle as it stands, on a bounded sample of the workload: last-mode slabs [0, slabs) sized to
    ~target_s of CPU work; when the whole tensor takes less, the whole-tensor sketch is repeated."""
    slabs = _calibrate_slabs(cfg, seed, om, target_s)
    t, f = _oracle_sample(cfg, seed, slabs, om)
    reps = 1
    if slabs == cfg.dims[-1] and t < 0.5 * target_s:
        reps = max(1, int(round(target_s / max(t, 1e-3))))
        t = sum(_oracle_sample(cfg, seed, slabs, om)[0] for _ in range(reps))
    return {"value": f * reps / t / 1e12, "unit": "TFLOP/s", "cores": _cores(), "kind": "oracle",
            "sample": f"fp64 numpy explicit-KR all-mode sketch of last-mode slabs [0,{slabs}) of {cfg.name} "
                      f"({slabs}/{cfg.dims[-1]} of the tensor) x{reps}, {t:.1f} s, os.cpu_count()={os.cpu_count()}"}


# ------------------------------------------------------------------ reference arm
def run_reference(args, cfg, rank, world):
    if rank != 0:
        return 0
    om = synth.omegas(cfg.dims, cfg.R, args.seed)
    budget = 150.0
    per_step = budget / max(1, args.steps + args.warmup)
    slabs = _calibrate_slabs(cfg, args.seed, om, per_step)
    for _ in range(args.warmup):
        _oracle_sample(cfg, args.seed, slabs, om)
    times, flops = [], 0
    for _ in range(args.steps):
        t, f = _oracle_sample(cfg, args.seed, slabs, om)
        times.append(t)
        flops = f
    tot = sum(times)
    value = flops * args.steps / tot / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _workload(cfg, world),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": _cores(), "kind": "oracle",
                         "sample": f"each step: fp64 oracle all-mode sketch of last-mode slabs [0,{slabs}) "
                                   f"of {cfg.name} ({slabs}/{cfg.dims[-1]} of the tensor)"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2507_23207_b200 as krp

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    Id = cfg.dims[-1]
    k0, kn = krp.krp_slab_range(Id, world, rank)  # the library's slab geometry
    k1 = k0 + kn
    dims_local = list(cfg.dims[:-1]) + [k1 - k0]
    n_local = int(np.prod(dims_local))
    x_host = torch.from_numpy(synth.tensor_slab(cfg, args.seed, k0, k1)).pin_memory()
    om_np = synth.omegas(cfg.dims, cfg.R, args.seed)
    om_host = [torch.from_numpy(o).pin_memory() for o in om_np]
    X = x_host.to(dev)
    om = [o.to(dev) for o in om_host]
    comm = krp.Comm() if world > 1 else None
    stream = torch.cuda.current_stream()

    if world > 1:
        ws = torch.empty(krp.krp_workspace_bytes_dist(krp.OP_SKETCH_ALL, dims_local, Id, cfg.R), dtype=torch.uint8,
                         device=dev)
        Y = [torch.empty((n, cfg.R), dtype=torch.float32, device=dev) for n in cfg.dims]

        def sketch():
            krp.krp_sketch_all_modes_dist(X, dims_local, Id, k0, om, comm, Y=Y, ws=ws)
    else:
        ws = torch.empty(krp.krp_workspace_bytes(krp.OP_SKETCH_ALL, cfg.dims, cfg.R), dtype=torch.uint8, device=dev)
        Y = [torch.empty((n, cfg.R), dtype=torch.float32, device=dev) for n in cfg.dims]

        def sketch():
            krp.krp_sketch_all_modes(X, cfg.dims, om, Y=Y, ws=ws)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, steps, sampler=None):
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if sampler:
            sampler.start()
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        clocks = sampler.stop() if sampler else None
        barrier()
        return max_over_ranks(e0.elapsed_time(e1)), clocks

    # ---- phase A: the headline all-mode sketch
    for _ in range(args.warmup):
        sketch()
    torch.cuda.synchronize()
    krp.krp_reset_launch_count()
    gpu_index = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local_rank)).split(",")[0]) \
        if os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")[0].isdigit() else local_rank
    t_ms, clocks = timed(sketch, args.steps, ClockSampler(gpu_index) if rank == 0 else None)
    launches = krp.krp_launch_count()
    # the dominant kernel's own duration: a second pass with CUDA events around each of its launches
    # (on the launching stream); kept out of the headline loop so the events do not perturb it
    krp.krp_profile_reset()
    krp.krp_profile_enable(True)
    timed(sketch, args.steps)
    krp.krp_profile_enable(False)
    k_ms, k_n, k_bytes, k_flops = krp.krp_profile_read()
    krp.krp_profile_reset()
    k_steps = args.steps
    flops_step = 4.0 * cfg.N * cfg.R
    value = flops_step * args.steps / (t_ms / 1e3) / 1e12

    # ---- roofline of the dominant kernel (algorithmic bytes / flops per launch over its event time)
    hbm_gbs, bf16_tf, peak_src = _peaks()
    tf32_tf = bf16_tf * (1.1 / 2.25)          # guide's nominal dense tf32 : bf16 ratio
    p3 = tf32_tf / 3.0                        # 3xTF32 split: three tf32 products per fp32 product
    t_hbm = 4.0 * cfg.N / (hbm_gbs * 1e9)
    t_tc = flops_step / (p3 * 1e12)
    bound = "hbm" if t_hbm >= t_tc else "tensor"
    avg_launch_s = (k_ms / 1e3) / max(k_n, 1)
    bytes_per_launch = k_bytes / max(k_n, 1)
    flops_per_launch = k_flops / max(k_n, 1)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        ent = tj.get(f"{cfg.name}:{world}") or tj.get(cfg.name)
        if ent:
            traffic = ent.get("dram_bytes_per_launch")
    if bound == "hbm":
        achieved = bytes_per_launch / avg_launch_s / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_gbs, "unit": "GB/s", "frac": achieved / hbm_gbs,
                "traffic": traffic}
    else:
        achieved = flops_per_launch / avg_launch_s / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": p3, "unit": "TFLOP/s", "frac": achieved / p3,
                "traffic": traffic}
    roof.update({"peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs burst; 3xTF32 = bf16 x 1.1/2.25 / 3)",
                 "kernel_ms_avg": 1e3 * avg_launch_s, "kernel_launches_per_step": k_n / k_steps,
                 "kernel_share_of_step": (k_ms / k_steps) / (t_ms / args.steps),
                 "roof_ms_step": 1e3 * max(t_hbm, t_tc)})

    # ---- phase B: full rHOSVD steps (sketch + QR + core + truncation)
    rhosvd_s = None
    rel_err = None
    if not args.no_rhosvd:
        if world > 1:
            wsr = torch.empty(krp.krp_workspace_bytes_dist(krp.OP_RHOSVD, dims_local, Id, cfg.R, cfg.ranks),
                              dtype=torch.uint8, device=dev)

            def rh(with_error=False):
                return krp.krp_rhosvd_dist(X, dims_local, Id, k0, cfg.ranks, om, comm, with_error=with_error,
                                           ws=None if with_error else wsr)
        else:
            wsr = torch.empty(krp.krp_workspace_bytes(krp.OP_RHOSVD, cfg.dims, cfg.R, cfg.ranks), dtype=torch.uint8,
                              device=dev)

            def rh(with_error=False):
                return krp.krp_rhosvd(X, cfg.dims, cfg.ranks, om, with_error=with_error,
                                      ws=None if with_error else wsr)
        for _ in range(min(args.warmup, 2)):
            rh()
        steps_b = max(1, min(args.steps, 10))
        tb, _ = timed(rh, steps_b)
        rhosvd_s = tb / 1e3 / steps_b
        del wsr
        rel_err = rh(with_error=True)[2]

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        Yh = [torch.empty((n, cfg.R), dtype=torch.float32).pin_memory() for n in cfg.dims]
        if world == 1:
            wsh = torch.empty(krp.krp_workspace_bytes(krp.OP_SKETCH_ALL_HOST, cfg.dims, cfg.R), dtype=torch.uint8,
                              device=dev)

            def e2e_step():
                krp.krp_sketch_all_modes_host(x_host, cfg.dims, om_host, Y=Yh, ws=wsh)
        else:
            def e2e_step():
                X.copy_(x_host, non_blocking=True)
                for o, oh in zip(om, om_host):
                    o.copy_(oh, non_blocking=True)
                krp.krp_sketch_all_modes_dist(X, dims_local, Id, k0, om, comm, Y=Y, ws=ws)
                for yh, y in zip(Yh, Y):
                    yh.copy_(y, non_blocking=True)
                torch.cuda.current_stream().synchronize()
        for _ in range(min(args.warmup, 2)):
            e2e_step()
        steps_e = max(1, min(args.steps, 10))
        te, _ = timed(e2e_step, steps_e)
        h2d = 4 * (int(np.prod(cfg.dims)) + sum(n * cfg.R for n in cfg.dims))
        d2h = 4 * sum(n * cfg.R for n in cfg.dims) * world
        e2e = {"value": flops_step * steps_e / (te / 1e3) / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": te / steps_e}
        if world == 1:
            del wsh

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args.seed, om_np)

    if comm is not None:
        comm.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Tucker/smooth tensors of BASELINE.json's configs; no dataset)",
            "config": _workload(cfg, world),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks, "rhosvd_s": rhosvd_s, "rhosvd_rel_err": rel_err,
            "pct_roofline": 100.0 * max(t_hbm, t_tc) / (t_ms / 1e3 / args.steps),
        }
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c2", choices=sorted(synth.CONFIGS))
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-rhosvd", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = synth.config(args.config)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return run_ours(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
