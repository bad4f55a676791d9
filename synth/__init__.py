"""Seeded synthetic inputs for the KRP-sketch path (shared by tests, bench and smoke).

This module holds NO arithmetic of the method (no sketch, no Khatri-Rao product,
no QR of a sketch, no core formation).  It only draws the random numbers and
builds the synthetic tensors that BASELINE.json's configs describe, so that the
fp64 oracle (``oracle/``) and the CUDA path (``paper_2507_23207_b200``) consume
bit-identical fp32 arrays.  Readings of the configs (R7/R9/R10/R11):

* Layout: a d-way tensor X with dims (I_1..I_d) is a flat fp32 buffer in
  first-index-fastest order (offset = sum_k i_k * prod_{m<k} I_m), i.e. the
  numpy array ``x.reshape(dims, order="F")``.  (SPEC S:28-33.)
* Generator: numpy PCG64 via ``default_rng([seed, tag, ...])``; fp64 draws,
  rounded once to fp32.  Tags: core 0, factor k -> 1+k, noise (100, i_d) per
  last-mode index (so a last-mode slab is identical whatever the sharding),
  Omega_k -> 200+k, STHOSVD step i / mode j -> (300, i, j).
* Noise: E iid N(0,1), scaled by eta * ||X0||_F / sqrt(N) (the expected norm of
  E), so each slab is generated independently.  ||X0||_F = ||core||_F for
  orthonormal factors.
* Decay "0.8^(i+j+k)" and the smooth function use 0-based indices.
* The paper's Cauchy tensor (NEXT-1): x = 1 / (i_1^a + ... + i_d^a)^(1/a) with 1-based
  indices, a = 2; closed form, no random numbers, no noise.  Computed in fp64 (integer powers,
  exact sums, a correctly rounded square root for a = 2) and rounded once to fp32, so the host generator
  here and the device generator (cauchy_device) give bit-identical tensors.
* "orthonormalised Gaussian factors": Q of a Householder QR of an iid N(0,1)
  I_k x r_k matrix.
"""
from __future__ import annotations

import dataclasses
import math
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "Config",
    "CONFIGS",
    "config",
    "rng",
    "omegas",
    "sthosvd_omegas",
    "tensor",
    "tensor_slab",
    "tucker_parts",
    "random_tensor",
    "cauchy_device",
    "rhosvd_fresh_omegas",
    "dense_gaussian",
    "dense_gaussian_sthosvd",
    "hadamard_tucker_inputs",
    "hadamard_omegas",
]


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    dims: Tuple[int, ...]
    R: int                       # sketch width l = r + p
    ranks: Tuple[int, ...]       # target Tucker ranks r_n
    kind: str                    # "tucker" | "smooth" | "cauchy"
    core: Tuple[int, ...] = ()   # Tucker core dims
    decay: Optional[float] = None  # core entry scale decay**(sum of 0-based indices)
    eta: float = 0.0             # relative noise level
    workload: str = "rhosvd"     # "rhosvd" | "sthosvd"
    alpha: float = 2.0           # Cauchy exponent (kind "cauchy")

    @property
    def d(self) -> int:
        return len(self.dims)

    @property
    def N(self) -> int:
        return int(np.prod(self.dims, dtype=np.int64))

    def scaled(self, dims: Sequence[int], name: Optional[str] = None) -> "Config":
        """Same recipe on smaller dims (core ranks clipped to the new dims)."""
        core = tuple(min(c, n) for c, n in zip(self.core, dims)) if self.core else ()
        ranks = tuple(min(r, n) for r, n in zip(self.ranks, dims))
        return dataclasses.replace(self, name=name or f"{self.name}@{'x'.join(map(str, dims))}",
                                   dims=tuple(int(n) for n in dims), core=core, ranks=ranks)


# BASELINE.json configs[0..4]
CONFIGS = {
    "c1": Config("c1", (64, 64, 64), 10, (5, 5, 5), "tucker", core=(5, 5, 5), eta=1e-4),
    "c2": Config("c2", (512, 512, 512), 40, (30, 30, 30), "tucker", core=(30, 30, 30), decay=0.8, eta=1e-3),
    "c3": Config("c3", (128, 128, 128, 128), 30, (20, 20, 20, 20), "tucker", core=(20, 20, 20, 20),
                 eta=1e-3, workload="sthosvd"),
    "c4": Config("c4", (64, 64, 64, 64, 64), 20, (10, 10, 10, 10, 10), "tucker", core=(10, 10, 10, 10, 10),
                 decay=0.7, eta=1e-4),
    "c5": Config("c5", (2048, 2048, 512), 60, (50, 50, 50), "smooth", eta=1e-6),
    # NEXT-1: the paper's 4-way Cauchy tensor, n = 250, a = 2, no oversampling (R = r);
    # the rank is swept by tools/cauchy_sweep.py, r = 30 here
    "cauchy": Config("cauchy", (250, 250, 250, 250), 30, (30, 30, 30, 30), "cauchy", workload="rhosvd"),
}


def config(name: str) -> Config:
    return CONFIGS[name]


def rng(seed: int, *tags: int) -> np.random.Generator:
    return np.random.default_rng([int(seed), *[int(t) for t in tags]])


def omegas(dims: Sequence[int], R: int, seed: int) -> List[np.ndarray]:
    """Memoized Omega_k in R^{I_k x R}, iid N(0,1), fp32, row-major (i*R + r)."""
    return [rng(seed, 200 + k).standard_normal((int(n), R)).astype(np.float32) for k, n in enumerate(dims)]


def sthosvd_omegas(dims: Sequence[int], R: int, seed: int) -> List[List[Optional[np.ndarray]]]:
    """Fresh set per STHOSVD step i: om[i][j] is I_j x R for j != i, None for j == i.

    For an already-compressed mode j < i only the leading r_j rows are read (R5)."""
    d = len(dims)
    return [[None if j == i else rng(seed, 300, i, j).standard_normal((int(dims[j]), R)).astype(np.float32)
             for j in range(d)] for i in range(d)]


def rhosvd_fresh_omegas(dims: Sequence[int], R: int, seed: int) -> List[List[Optional[np.ndarray]]]:
    """Alg. 7 read literally (NEXT-2): a fresh set per mode n, om[n][j] is I_j x R (j != n).
    Tags (400, n, j)."""
    d = len(dims)
    return [[None if j == n else rng(seed, 400, n, j).standard_normal((int(dims[j]), R)).astype(np.float32)
             for j in range(d)] for n in range(d)]


def dense_gaussian(dims: Sequence[int], R: int, seed: int) -> List[np.ndarray]:
    """Dense Gaussian test matrices of the RHOSVD baseline (Table 1): Omega_n is (N / I_n) x R, iid N(0,1),
    fp32, row-major, rows in the column order of X_(n).  Tags (500, n)."""
    N = int(np.prod(dims))
    return [rng(seed, 500, n).standard_normal((N // int(dims[n]), R)).astype(np.float32) for n in range(len(dims))]


def dense_gaussian_sthosvd(dims: Sequence[int], ranks: Sequence[int], R: int, seed: int) -> List[np.ndarray]:
    """Dense Gaussian test matrices of the RSTHOSVD baseline: step i sketches the current core (modes j < i already
    compressed to r_j), Omega_i is (prod_{j<i} r_j prod_{j>i} I_j) x R.  Tags (600, i)."""
    out = []
    for i in range(len(dims)):
        rows = int(np.prod([ranks[j] for j in range(i)] + [dims[j] for j in range(i + 1, len(dims))]))
        out.append(rng(seed, 600, i).standard_normal((rows, R)).astype(np.float32))
    return out


def hadamard_tucker_inputs(ns: Sequence[int], qs: Sequence[int], ss: Sequence[int], seed: int):
    """Two 3-way Tucker tensors X = F ×_n A_n (cores q) and Y = G ×_n U_n (cores s) with iid N(0,1) cores and
    orthonormalised Gaussian factors (the App. C setting), fp32.  Tags (700, ...)."""
    f = rng(seed, 700).standard_normal(tuple(qs)).astype(np.float32)
    g = rng(seed, 701).standard_normal(tuple(ss)).astype(np.float32)
    xs = [np.linalg.qr(rng(seed, 702, k).standard_normal((n, q)))[0].astype(np.float32) for k, (n, q) in enumerate(zip(ns, qs))]
    ys = [np.linalg.qr(rng(seed, 703, k).standard_normal((n, q)))[0].astype(np.float32) for k, (n, q) in enumerate(zip(ns, ss))]
    return f, xs, g, ys


def hadamard_omegas(ns: Sequence[int], ls: Sequence[int], seed: int) -> List[List[Optional[np.ndarray]]]:
    """Ω_{i,j} ∈ R^{n_j x l_i} (Alg. 9 line 2), iid N(0,1), fp32; None on the diagonal.  Tags (710, i, j)."""
    d = len(ns)
    return [[None if j == i else rng(seed, 710, i, j).standard_normal((int(ns[j]), int(ls[i]))).astype(np.float32)
             for j in range(d)] for i in range(d)]


def _orth_factor(n: int, r: int, seed: int, k: int) -> np.ndarray:
    g = rng(seed, 1 + k).standard_normal((n, r))
    q, _ = np.linalg.qr(g)
    return q


def tucker_parts(cfg: Config, seed: int):
    """(core fp64 Fortran-ordered, [U_k fp64], ||X0||_F) of a Tucker config."""
    assert cfg.kind == "tucker"
    core = rng(seed, 0).standard_normal(int(np.prod(cfg.core))).reshape(cfg.core, order="F")
    if cfg.decay is not None:
        idx = np.indices(cfg.core).sum(axis=0)
        core = core * cfg.decay ** idx
    us = [_orth_factor(n, r, seed, k) for k, (n, r) in enumerate(zip(cfg.dims, cfg.core))]
    return core, us, float(np.linalg.norm(core))


def _smooth_norm(dims: Sequence[int]) -> float:
    i1, i2, i3 = dims
    a = (np.arange(i1)[:, None] / i1 + np.arange(i2)[None, :] / i2).ravel()
    vals, cnt = np.unique(a, return_counts=True)
    tot = 0.0
    for k in range(i3):
        tot += float(np.sum(cnt / (1.0 + vals + k / i3) ** 2))
    return math.sqrt(tot)


def _cauchy_slab(dims: Sequence[int], alpha: float, k0: int, k1: int) -> np.ndarray:
    """Cauchy tensor slab x[..., k0:k1] = 1 / (sum_j i_j^a)^(1/a), 1-based indices, fp64."""
    d = len(dims)
    s = np.zeros(tuple(dims[:-1]) + (k1 - k0,))
    for j in range(d):
        idx = np.arange(1, dims[j] + 1, dtype=np.float64) if j < d - 1 else np.arange(k0 + 1, k1 + 1, dtype=np.float64)
        shape = [1] * d
        shape[j] = idx.size
        s = s + (idx * idx if alpha == 2.0 else idx ** alpha).reshape(shape)
    return np.asfortranarray(1.0 / (np.sqrt(s) if alpha == 2.0 else s ** (1.0 / alpha)))


def cauchy_device(dims: Sequence[int], alpha: float = 2.0, device="cuda"):
    """The Cauchy tensor generated on the device with torch (the same fp64 formula as _cauchy_slab, rounded once
    to fp32): a flat first-index-fastest fp32 tensor.  For the full n = 250 workload (15.6 GB), which is too
    large to build on the host in reasonable time."""
    import torch
    d = len(dims)
    out = torch.empty(int(np.prod(dims)), dtype=torch.float32, device=device)
    inner = int(np.prod(dims[:-1]))
    # sum over the first d-1 modes of i_j^a, first index fastest (fp64: exact integers)
    s = torch.zeros(inner, dtype=torch.float64, device=device)
    stride = 1
    for j in range(d - 1):
        idx = torch.arange(inner, device=device, dtype=torch.int64) // stride % dims[j] + 1
        v = idx.to(torch.float64)
        s += v * v if alpha == 2.0 else v ** alpha
        stride *= dims[j]
    for k in range(dims[-1]):
        kk = float((k + 1) * (k + 1)) if alpha == 2.0 else float(k + 1) ** alpha
        t = s + kk
        out[k * inner:(k + 1) * inner] = (1.0 / (torch.sqrt(t) if alpha == 2.0 else t ** (1.0 / alpha))).to(torch.float32)
    return out


def _x0_slab(cfg: Config, seed: int, k0: int, k1: int, parts=None) -> np.ndarray:
    """Noise-free fp64 slab X0[..., k0:k1] (Fortran-ordered array of dims[:-1] + (k1-k0,))."""
    dims = cfg.dims
    if cfg.kind == "cauchy":
        return _cauchy_slab(dims, cfg.alpha, k0, k1)
    if cfg.kind == "smooth":
        assert cfg.d == 3
        i1, i2, i3 = dims
        a = np.arange(i1)[:, None, None] / i1 + np.arange(i2)[None, :, None] / i2
        k = np.arange(k0, k1)[None, None, :] / i3
        return np.asfortranarray(1.0 / (1.0 + a + k))
    core, us, _ = parts if parts is not None else tucker_parts(cfg, seed)
    t = core
    # contract the last mode first with the slab rows, then the others (data generation only)
    ul = us[-1][k0:k1]
    t = np.tensordot(t, ul, axes=([cfg.d - 1], [1]))  # dims core[:-1] + (slab,)
    for m in range(cfg.d - 1):
        t = np.tensordot(t, us[m], axes=([0], [1]))  # rotates axes: contracted axis appended last
    # after d-1 rotations the axis order is (slab, I_1, ..., I_{d-1}); move slab to the end
    t = np.moveaxis(t, 0, -1)
    return np.asfortranarray(t)


def x0_norm(cfg: Config, seed: int, parts=None) -> float:
    if cfg.kind == "cauchy":
        return 0.0  # no noise is added (the norm only scales the noise)
    if cfg.kind == "smooth":
        return _smooth_norm(cfg.dims)
    return (parts if parts is not None else tucker_parts(cfg, seed))[2]


def tensor_slab(cfg: Config, seed: int, k0: int, k1: int, parts=None, xnorm=None) -> np.ndarray:
    """fp32 slab X[..., k0:k1] as a flat first-index-fastest buffer of length N/I_d*(k1-k0)."""
    if parts is None and cfg.kind == "tucker":
        parts = tucker_parts(cfg, seed)
    if xnorm is None:
        xnorm = x0_norm(cfg, seed, parts)
    inner = int(np.prod(cfg.dims[:-1]))
    out = np.empty(inner * (k1 - k0), dtype=np.float32)
    scale = cfg.eta * xnorm / math.sqrt(cfg.N) if cfg.eta else 0.0
    step = max(1, (1 << 22) // max(inner, 1))  # chunk boundaries at global multiples of step: any slab
                                                # request reproduces the whole tensor's bits

    def fill(s0):
        # each chunk of last-mode indices is independent (its own noise streams), so chunks are generated
        # on a thread pool (numpy releases the GIL)
        s1 = min(k1, (s0 // step + 1) * step)
        x0 = _x0_slab(cfg, seed, s0, s1, parts).reshape(-1, order="F")
        if scale:
            noise = np.concatenate([rng(seed, 100, kk).standard_normal(inner) for kk in range(s0, s1)])
            x0 = x0 + scale * noise
        out[(s0 - k0) * inner:(s1 - k0) * inner] = x0.astype(np.float32)

    starts = [k0] + list(range((k0 // step + 1) * step, k1, step))
    if len(starts) > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=min(len(starts), os.cpu_count() or 1)) as ex:
            list(ex.map(fill, starts))
    else:
        for s0 in starts:
            fill(s0)
    return out


def tensor(cfg: Config, seed: int) -> np.ndarray:
    """Whole fp32 tensor, flat first-index-fastest."""
    return tensor_slab(cfg, seed, 0, cfg.dims[-1])


def random_tensor(dims: Sequence[int], seed: int, tag: int = 7) -> np.ndarray:
    """iid N(0,1) fp32 tensor (flat, first-index-fastest) for edge-case / ragged tests."""
    return rng(seed, 900, tag).standard_normal(int(np.prod(dims))).astype(np.float32)
