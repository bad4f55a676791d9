#!/usr/bin/env python
"""bench.py — all-mode KRP sketch throughput (and rHOSVD time) on B200, BASELINE.json's metric.

Default (N=1): BASELINE configs[4] = c5, the largest single-GPU config (2048 x 2048 x 512 fp32 smooth
tensor + 1e-6 noise, R = 60, 8 GiB resident in HBM: larger than L2, no flush needed), the tensor the
8-GPU scaling target names.  Inputs under 2x L2 (c1) are flushed between timed steps.  The same line
carries per-config kernel fractions for c2-c5 ("per_config") and the c3 STHOSVD time.

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
    """Number of last-mode slabs whose oracle sketch takes about target_s.  The oracle's time is affine in
    the slab count (forming the explicit Khatri-Rao matrix of the last mode's sketch costs the same for any
    slab), so two samples fit t = a + b * slabs; a proportional fit would stop at a sample that is almost all
    fixed cost (c5: 3 of 512 slabs)."""
    Id = cfg.dims[-1]
    s1, t1 = 1, 0.0
    while s1 < Id:
        t1, _ = _oracle_sample(cfg, seed, s1, om)
        if t1 >= 0.25 * target_s:
            break
        s1 = min(Id, s1 * 2)
    if s1 >= Id or t1 <= 0 or t1 >= target_s:
        return int(max(1, min(Id, s1 * target_s / t1))) if t1 > 0 else s1
    s2 = min(Id, max(s1 + 1, 4 * s1))
    t2, _ = _oracle_sample(cfg, seed, s2, om)
    b = max((t2 - t1) / (s2 - s1), 0.01 * t1 / s1)  # floor: a noisy pair must not extrapolate without bound
    a = max(t1 - b * s1, 0.0)
    return int(max(1, min(Id, (target_s - a) / b)))


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
def _roofline(cfg_dims, R, k_ms, k_n, k_bytes, k_flops, steps):
    """Roofline of the dominant sketch kernel: algorithmic bytes (4 B per element, X read once) or flops
    (4NR) per launch over its CUDA-event duration, against MEASURED_PEAKS.json."""
    N = float(np.prod(cfg_dims))
    hbm_gbs, bf16_tf, peak_src = _peaks()
    p3 = bf16_tf * (1.1 / 2.25) / 3.0  # tf32 = bf16 x nominal 1.1/2.25; 3xTF32 = three tf32 products
    t_hbm = 4.0 * N / (hbm_gbs * 1e9)
    t_tc = 4.0 * N * R / (p3 * 1e12)
    bound = "hbm" if t_hbm >= t_tc else "tensor"
    avg_s = (k_ms / 1e3) / max(k_n, 1)
    if bound == "hbm":
        achieved = (k_bytes / max(k_n, 1)) / avg_s / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_gbs, "unit": "GB/s", "frac": achieved / hbm_gbs}
    else:
        achieved = (k_flops / max(k_n, 1)) / avg_s / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": p3, "unit": "TFLOP/s", "frac": achieved / p3}
    roof.update({"peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs / bf16_tflops burst; "
                                f"3xTF32 = bf16 x 1.1/2.25 / 3)",
                 "kernel_ms_avg": 1e3 * avg_s, "kernel_launches_per_step": k_n / max(steps, 1),
                 "roof_ms": 1e3 * max(t_hbm, t_tc)})
    return roof


def _traffic(name, world):
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        # a capture is per launch of one GPU's kernel: the whole-tensor entry holds for N = 1 only (a rank's
        # slab launch moves 1/N of it); N > 1 needs its own "<cfg>:<N>" entry, else traffic is null
        ent = tj.get(f"{name}:{world}") or (tj.get(name) if world == 1 else None)
        if ent:
            return ent.get("dram_bytes_per_launch")
    return None


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
    x_host = torch.from_numpy(synth.tensor_slab(cfg, args.seed, k0, k1)).pin_memory()
    om_np = synth.omegas(cfg.dims, cfg.R, args.seed)
    om_host = [torch.from_numpy(o).pin_memory() for o in om_np]
    X = x_host.to(dev)
    om = [o.to(dev) for o in om_host]
    comm = krp.Comm() if world > 1 else None
    stream = torch.cuda.current_stream()
    l2_bytes = int(getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 126 * 2 ** 20))
    # inputs smaller than twice the L2 are flushed between timed steps (a write of 2x L2, outside the events)
    flush = 4 * int(np.prod(dims_local)) < 2 * l2_bytes
    flush_buf = torch.empty(2 * l2_bytes // 4, dtype=torch.float32, device=dev) if flush else None

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

    def timed(fn, steps, sampler=None, flush_l2=False):
        """Device time of `steps` calls (CUDA events on the launching stream), max over ranks.  With flush_l2
        every step is bracketed by its own events and preceded (outside them) by a 2x-L2 write."""
        barrier()
        torch.cuda.synchronize()
        if sampler:
            sampler.start()
        if flush_l2:
            evs = []
            for _ in range(steps):
                flush_buf.fill_(1.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fn()
                e1.record(stream)
                evs.append((e0, e1))
            torch.cuda.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in evs)
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
        clocks = sampler.stop() if sampler else None
        barrier()
        return max_over_ranks(ms), clocks

    def timed_profiled(fn, steps, sampler=None, flush_l2=False):
        """timed() with the library profiler on: CUDA events on the launching stream around every launch of
        the dominant kernel INSIDE the timed region (so the kernel time and the step time see the same clocks
        and power state).  Returns (step ms, clocks, (kernel ms, launches, alg bytes, alg flops))."""
        krp.krp_profile_reset()
        krp.krp_profile_enable(True)
        ms, clocks = timed(fn, steps, sampler, flush_l2=flush_l2)
        krp.krp_profile_enable(False)
        r = krp.krp_profile_read()
        krp.krp_profile_reset()
        return ms, clocks, r

    # ---- phase A: the headline all-mode sketch
    for _ in range(args.warmup):
        sketch()
    torch.cuda.synchronize()
    krp.krp_reset_launch_count()
    gpu_index = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local_rank)).split(",")[0]) \
        if os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")[0].isdigit() else local_rank
    # the dominant kernel's own duration: CUDA events around each of its launches on the launching stream,
    # recorded inside the timed region (a separate pass ran later, hotter, and read the kernel longer than
    # the step it belongs to: r02d/r02f kernel_share_of_step 1.07-1.08 at c5)
    t_ms, clocks, (k_ms, k_n, k_bytes, k_flops) = timed_profiled(
        sketch, args.steps, ClockSampler(gpu_index) if rank == 0 else None, flush_l2=flush)
    launches = krp.krp_launch_count()
    flops_step = 4.0 * cfg.N * cfg.R
    value = flops_step * args.steps / (t_ms / 1e3) / 1e12
    roof = _roofline(dims_local, cfg.R, k_ms, k_n, k_bytes, k_flops, args.steps)
    roof["traffic"] = _traffic(cfg.name, world)
    roof["kernel_share_of_step"] = (k_ms / args.steps) / (t_ms / args.steps)

    # ---- phase B: full rHOSVD steps (sketch + QR + core + truncation) on the headline tensor
    rhosvd_s = None
    rel_err = None
    rh_clocks = None
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
        torch.cuda.synchronize()
        time.sleep(1.0)  # power-budget recovery after phase A (its clocks are sampled and reported either way)
        tb, rh_clocks = timed(rh, steps_b, ClockSampler(gpu_index) if rank == 0 else None)
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
        steps_e = max(1, min(args.steps, 5))
        te, _ = timed(e2e_step, steps_e)
        h2d = 4 * (int(np.prod(dims_local)) + sum(n * cfg.R for n in cfg.dims))
        d2h = 4 * sum(n * cfg.R for n in cfg.dims)
        e2e = {"value": flops_step * steps_e / (te / 1e3) / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d * world,
               "d2h_bytes_per_step": d2h * world, "ms_per_step": te / steps_e}
        if world == 1:
            del wsh

    # ---- per-config kernel fractions (c2-c5, and STHOSVD time on c3), rank 0 at N = 1: N(0,1) device data of
    # each config's shape (the sketch's time does not depend on the values), the same kernel profiler
    per_config = None
    if rank == 0 and world == 1 and not args.no_per_config:
        per_config = {}
        gen = torch.Generator(device=dev)
        gen.manual_seed(1234)
        for name in ("c2", "c3", "c4", "c5"):
            c = synth.config(name)
            if name == cfg.name:
                Xc, omc = X, om
            else:
                Xc = torch.randn(c.N, generator=gen, device=dev, dtype=torch.float32)
                omc = [torch.randn((n, c.R), generator=gen, device=dev, dtype=torch.float32) for n in c.dims]
            Yc = [torch.empty((n, c.R), dtype=torch.float32, device=dev) for n in c.dims]
            wsc = torch.empty(krp.krp_workspace_bytes(krp.OP_SKETCH_ALL, c.dims, c.R), dtype=torch.uint8, device=dev)

            def sk(Xc=Xc, omc=omc, Yc=Yc, wsc=wsc, c=c):
                krp.krp_sketch_all_modes(Xc, c.dims, omc, Y=Yc, ws=wsc)
            for _ in range(3):
                sk()
            nst = 10
            torch.cuda.synchronize()
            time.sleep(1.0)  # let the board's power budget recover after the previous phase (c5 runs power-capped)
            tms, pclk, kr = timed_profiled(sk, nst, ClockSampler(gpu_index) if rank == 0 else None)
            rf = _roofline(c.dims, c.R, *kr, nst)
            entry = {"dims": list(c.dims), "R": c.R, "step_ms": tms / nst, "tflops_step": 4.0 * c.N * c.R / (tms / nst / 1e3) / 1e12,
                     "bound": rf["bound"], "achieved": rf["achieved"], "unit": rf["unit"], "frac": rf["frac"],
                     "kernel_ms_avg": rf["kernel_ms_avg"], "roof_ms": rf["roof_ms"], "traffic": _traffic(name, 1),
                     "data": "N(0,1) device data of the config's shape" if name != cfg.name else "the headline tensor",
                     "clocks": pclk}
            if name == "c3":  # the c3 workload is STHOSVD (Alg. 8)
                oms3 = synth.sthosvd_omegas(c.dims, c.R, 0)
                dom = [[None if o is None else torch.from_numpy(o).to(dev) for o in row] for row in oms3]
                wss = torch.empty(krp.krp_workspace_bytes(krp.OP_STHOSVD, c.dims, c.R, c.ranks), dtype=torch.uint8,
                                  device=dev)

                def st(Xc=Xc, dom=dom, wss=wss, c=c):
                    krp.krp_sthosvd(Xc, c.dims, c.ranks, dom, ws=wss)
                st()
                ts_, _ = timed(st, 3)
                entry["sthosvd_s"] = ts_ / 1e3 / 3
                del wss
            per_config[name] = entry
            del Yc, wsc
            if name != cfg.name:
                del Xc, omc
            torch.cuda.empty_cache()

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args.seed, om_np)

    if comm is not None:
        comm.close()
    if rank == 0:
        wl = _workload(cfg, world)
        wl["l2"] = ("inputs smaller than 2x L2: a 2x-L2 write between timed steps, outside the step events"
                    if flush else "inputs larger than 2x L2 (no flush needed)")
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Tucker/smooth tensors of BASELINE.json's configs; no dataset)",
            "config": wl, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks, "rhosvd_s": rhosvd_s, "rhosvd_rel_err": rel_err, "rhosvd_clocks": rh_clocks,
            "per_config": per_config,
        }
        print(json.dumps(line), flush=True)
    return 0


def _free_port():
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    return port


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c5", choices=sorted(synth.CONFIGS))
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-rhosvd", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-config", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = synth.config(args.config)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # launched without torchrun: start one rank per GPU ourselves (same arguments), rank 0 prints the line
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        return 2
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
