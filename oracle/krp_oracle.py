"""fp64 CPU oracle for randomized HOSVD / STHOSVD with Khatri-Rao products.

TEST INFRASTRUCTURE.  Plain, slow, obviously-correct numpy (fp64) versions of
every step of the hot path, written from PAPER.md (arXiv 2507.23207) and cited
line by line (``P:n`` = line n of PAPER.md).  It shares no code with the CUDA
path and must only be used by tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline / reference legs.

Conventions (DESIGN.md §3 readings):
* Tensors are numpy arrays indexed ``x[i_1, ..., i_d]`` whose flat storage is
  first-index-fastest: ``x = flat.reshape(dims, order="F")`` (R1).
* The mode-n unfolding X_(n) is I_n x prod_{k!=n} I_k with column index
  sum_{k!=n} i_k J_k, J_k = prod_{m<k, m!=n} I_m.  Then
  (Omega_d ⊙ ... ⊙ Omega_{n+1} ⊙ Omega_{n-1} ⊙ ... ⊙ Omega_1) has its rows in
  exactly that column order, which is the pairing under which
  the MTTKRP of Alg. 7 line 3 is the plain matrix product below.
* Inputs arrive as fp32 and are upcast to fp64 once.
* Memory-only chunking: a sum over the columns of X_(n) may be split into
  consecutive last-mode index ranges (``chunk``); this changes only the fp64
  rounding order, never the terms.  ``chunk=None`` is the unsplit product.

Parity status of each function is recorded in DESIGN.md §4 ("pins"); every
function here is pinned by a test in tests/test_oracle_pins.py.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "as_tensor",
    "unfold",
    "fold",
    "kron",
    "khatri_rao",
    "kr_for_mode",
    "sketch_mode",
    "sketch_all_modes",
    "sketch_mode_rows",
    "sketch_rows_ttv",
    "thin_qr",
    "ttm",
    "multi_ttm",
    "leading_left_singular_vectors", "canonical_signs",
    "rhosvd",
    "sthosvd",
    "reconstruct",
    "tucker_error",
    "sketch_flops",
    "hosvd",
    "sthosvd_deterministic",
    "rhosvd_fresh",
    "rhosvd_gaussian",
    "sthosvd_gaussian",
    "row_kron",
    "hadamard_tucker_explicit",
    "hadamard_tucker_rhosvd",
]


# ----------------------------------------------------------------- tensor algebra
def as_tensor(flat: np.ndarray, dims: Sequence[int]) -> np.ndarray:
    """fp32/fp64 flat first-index-fastest buffer -> fp64 array x[i_1..i_d]."""
    return np.asarray(flat, dtype=np.float64).reshape(tuple(int(n) for n in dims), order="F")


def unfold(x: np.ndarray, n: int) -> np.ndarray:
    """Mode-n unfolding X_(n): rows i_n, columns = remaining indices,
    first remaining index fastest."""
    return np.moveaxis(x, n, 0).reshape(x.shape[n], -1, order="F")


def fold(m: np.ndarray, n: int, dims: Sequence[int]) -> np.ndarray:
    """Inverse of ``unfold``."""
    dims = tuple(int(v) for v in dims)
    rest = dims[:n] + dims[n + 1:]
    return np.moveaxis(m.reshape((dims[n],) + rest, order="F"), 0, n)


def kron(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Kronecker product, block matrix [a_ij * B]."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    m, n = a.shape
    p, q = b.shape
    out = np.empty((m * p, n * q))
    for i in range(m):
        for j in range(n):
            out[i * p:(i + 1) * p, j * q:(j + 1) * q] = a[i, j] * b
    return out


def khatri_rao(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Khatri-Rao (column-wise Kronecker) product: column r = a_r ⊗ b_r."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape[1] == b.shape[1]
    return np.stack([np.kron(a[:, r], b[:, r]) for r in range(a.shape[1])], axis=1)


def kr_for_mode(omegas: Sequence[np.ndarray], n: int) -> np.ndarray:
    """Omega_d ⊙ ... ⊙ Omega_{n+1} ⊙ Omega_{n-1} ⊙ ... ⊙ Omega_1 (Alg. 7 line 3).

    Formed explicitly, left to right in the paper's order."""
    others = [np.asarray(omegas[k], dtype=np.float64) for k in range(len(omegas) - 1, -1, -1) if k != n]
    w = others[0]
    for o in others[1:]:
        w = khatri_rao(w, o)
    return w


# ----------------------------------------------------------------- the sketch (MTTKRP)
def _slab_ranges(last: int, chunk: Optional[int]):
    if chunk is None or chunk >= last:
        return [(0, last)]
    return [(k, min(last, k + chunk)) for k in range(0, last, chunk)]


def sketch_mode(x: np.ndarray, omegas: Sequence[np.ndarray], n: int, chunk: Optional[int] = None) -> np.ndarray:
    """Y_n = X_(n) (Omega_d ⊙ ... ⊙ Omega_{n+1} ⊙ Omega_{n-1} ⊙ ... ⊙ Omega_1)
    (Alg. 7 line 3; BASELINE north_star), explicit KR times the unfolding.

    ``x`` is the fp64 tensor x[i_1..i_d]; ``omegas[k]`` is I_k x R (omegas[n] unused).
    With ``chunk``, the columns of X_(n) are taken in last-mode slabs: for n < d-1
    the slab products are summed, for n = d-1 each slab fills its own rows."""
    d = x.ndim
    R = np.asarray(omegas[(n + 1) % d]).shape[1]
    last = x.shape[-1]
    if n == d - 1:
        w = kr_for_mode(omegas, n)  # does not involve Omega_d
        y = np.zeros((x.shape[n], R))
        for k0, k1 in _slab_ranges(last, chunk):
            y[k0:k1] = unfold(x[..., k0:k1], n) @ w
        return y
    y = np.zeros((x.shape[n], R))
    for k0, k1 in _slab_ranges(last, chunk):
        om = list(omegas)
        om[d - 1] = np.asarray(omegas[d - 1])[k0:k1]
        y += unfold(x[..., k0:k1], n) @ kr_for_mode(om, n)
    return y


def sketch_all_modes(x: np.ndarray, omegas: Sequence[np.ndarray], chunk: Optional[int] = None) -> List[np.ndarray]:
    """Memoized sketches: one shared set {Omega_k} reused for every mode."""
    return [sketch_mode(x, omegas, n, chunk) for n in range(x.ndim)]


def sketch_mode_rows(flat: np.ndarray, dims: Sequence[int], omegas: Sequence[np.ndarray], n: int,
                     rows: Sequence[int]) -> np.ndarray:
    """Rows ``rows`` of Y_n only (sampled full-size parity): Y_n(i,:) = X_(n)(i,:) · KR_n,
    with X_(n)(i,:) gathered from the fp32 buffer one last-mode slab at a time."""
    dims = tuple(int(v) for v in dims)
    d = len(dims)
    R = np.asarray(omegas[(n + 1) % d]).shape[1]
    inner = int(np.prod(dims[:-1]))
    out = np.zeros((len(rows), R))
    if n == d - 1:
        w = kr_for_mode(omegas, n)
        for t, i in enumerate(rows):
            out[t] = np.asarray(flat[i * inner:(i + 1) * inner], dtype=np.float64) @ w
        return out
    w_in = kr_for_mode([o for o in omegas[:-1]] + [np.ones((1, R))], n)  # modes < d except n
    for k in range(dims[-1]):
        slab = as_tensor(flat[k * inner:(k + 1) * inner], dims[:-1])
        xu = unfold(slab, n)  # I_n x prod_{m<d-1, m!=n} I_m
        for t, i in enumerate(rows):
            out[t] += (xu[i] @ w_in) * np.asarray(omegas[d - 1][k], dtype=np.float64)
    return out


def sketch_rows_ttv(flat: np.ndarray, dims: Sequence[int], omegas: Sequence[np.ndarray], n: int,
                    rows: Sequence[int]) -> np.ndarray:
    """Rows ``rows`` of Y_n by the column identity Y_n(i, j) = (X ×_{k≠n} ω_k^(j)ᵀ)(i)  (column
    j of Ω_d ⊙ ⋯ ⊙ Ω_1 is ω_d^(j) ⊗ ⋯ ⊗ ω_1^(j), so the MTTKRP column is a multi-TTV).

    For each requested i it gathers the sub-tensor X(i_n = i) from the flat fp32 buffer (no full fp64
    copy of X) and contracts the remaining modes one at a time, keeping the column index j diagonal:
    T(j, ...) <- Σ_{i_k} T(j, i_k, ...) Ω_k(i_k, j).  Used for sampled parity at full BASELINE sizes,
    where the explicit Khatri-Rao product does not fit in memory."""
    dims = tuple(int(v) for v in dims)
    d = len(dims)
    R = np.asarray(omegas[(n + 1) % d]).shape[1]
    x = np.asarray(flat).reshape(dims[::-1])  # C-order view: axis a holds mode d-1-a (first index fastest)
    out = np.zeros((len(rows), R))
    others = [k for k in range(d) if k != n]
    for t, i in enumerate(rows):
        sub = np.asarray(np.take(x, int(i), axis=d - 1 - n), dtype=np.float64)  # axes: modes others[::-1]
        # contract the slowest remaining mode first (leading axis), keeping j as the leading axis
        k = others[-1]
        T = np.einsum("a...,aj->j...", sub, np.asarray(omegas[k], dtype=np.float64))
        for k in others[-2::-1]:
            T = np.einsum("ja...,aj->j...", T, np.asarray(omegas[k], dtype=np.float64))
        out[t] = T
    return out


# ----------------------------------------------------------------- orthonormalisation, TTM
def thin_qr(y: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """Thin QR Y = Q R (Alg. 1 line 3; Alg. 7 line 4) by Householder
    (LAPACK geqrf via numpy), columns signed so that diag(R) > 0 (the unique Q of a
    full-rank Y, the one CholeskyQR also produces)."""
    q, r = np.linalg.qr(np.asarray(y, dtype=np.float64), mode="reduced")
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return q * s[None, :], r * s[:, None]


def ttm(x: np.ndarray, a: np.ndarray, n: int) -> np.ndarray:
    """Tensor-times-matrix Y = X ×_n A, i.e. Y_(n) = A X_(n)."""
    dims = list(x.shape)
    dims[n] = a.shape[0]
    return fold(np.asarray(a, dtype=np.float64) @ unfold(x, n), n, dims)


def multi_ttm(x: np.ndarray, mats: Sequence[Optional[np.ndarray]]) -> np.ndarray:
    """X ×_1 A_1 ×_2 ... ×_d A_d, applied in ascending mode order (None = identity)."""
    y = x
    for n, a in enumerate(mats):
        if a is not None:
            y = ttm(y, a, n)
    return y


def canonical_signs(u: np.ndarray) -> np.ndarray:
    """Columns signed so that each column's entry of largest magnitude (first on ties) is positive
    (reading R24: singular vectors are defined up to sign; STHOSVD's later sketches
    pair the rows of Omega_j with the basis chosen at step j (R5), so both sides fix the sign the
    same way)."""
    u = np.array(u, dtype=np.float64, copy=True)
    for t in range(u.shape[1]):
        i = int(np.argmax(np.abs(u[:, t])))
        if u[i, t] < 0:
            u[:, t] = -u[:, t]
    return u


def leading_left_singular_vectors(m: np.ndarray, r: int) -> Tuple[np.ndarray, np.ndarray]:
    """U(:, 1:r) and the singular values of M (LAPACK SVD), Alg. 2 line 2-3 pattern, signs
    canonical (reading R24)."""
    u, s, _ = np.linalg.svd(np.asarray(m, dtype=np.float64), full_matrices=False)
    return canonical_signs(u[:, :r]), s


# ----------------------------------------------------------------- Tucker algorithms
def _core_slabwise(x: np.ndarray, qs: Sequence[np.ndarray], chunk: Optional[int]) -> np.ndarray:
    """G = X ×_1 Q_1ᵀ ×_2 ... ×_d Q_dᵀ (Alg. 7 line 6), last-mode slabs summed."""
    d = x.ndim
    g = None
    for k0, k1 in _slab_ranges(x.shape[-1], chunk):
        mats = [q.T for q in qs[:-1]] + [qs[-1][k0:k1].T]
        part = multi_ttm(x[..., k0:k1], mats)
        g = part if g is None else g + part
    return g


def reconstruct(core: np.ndarray, qs: Sequence[np.ndarray]) -> np.ndarray:
    """X̂ = G ×_1 Q_1 ×_2 ... ×_d Q_d."""
    return multi_ttm(core, list(qs))


def tucker_error(x: np.ndarray, core: np.ndarray, qs: Sequence[np.ndarray], chunk: Optional[int] = None) -> float:
    """||X - X̂||_F / ||X||_F, X̂ rebuilt slab by slab."""
    num = 0.0
    den = 0.0
    for k0, k1 in _slab_ranges(x.shape[-1], chunk):
        xh = multi_ttm(core, list(qs[:-1]) + [qs[-1][k0:k1]])
        diff = x[..., k0:k1] - xh
        num += float(np.sum(diff * diff))
        den += float(np.sum(x[..., k0:k1] ** 2))
    return float(np.sqrt(num / den))


def rhosvd(x: np.ndarray, omegas: Sequence[np.ndarray], ranks: Sequence[int], chunk: Optional[int] = None,
           with_error: bool = True):
    """RHOSVD-KRP-MEMO (Alg. 7 with memoization) + truncation R4.

    1. Y_n = MTTKRP with the shared {Omega_k}       for every n
    2. Q_n = thin QR of Y_n, diag(R) > 0                    (l_n = R columns)
    3. G = X ×_1 Q_1ᵀ ... ×_d Q_dᵀ
    4. if r_n < l_n: U_n = leading r_n left singular vectors of G_(n) of the untruncated core
       (HOSVD of the core: "hosvd on the core", Alg. 2 pattern P:118-120); Q_n <- Q_n U_n;
       then G <- G ×_1 U_1ᵀ ... ×_d U_dᵀ
    5. relative error ||X - [G; Q]|| / ||X||
    Returns (qs, core, err, ys)."""
    return _rhosvd_from_sketches(x, sketch_all_modes(x, omegas, chunk), ranks, chunk, with_error)


def _rhosvd_from_sketches(x: np.ndarray, ys: Sequence[np.ndarray], ranks: Sequence[int], chunk: Optional[int],
                          with_error: bool):
    """Alg. 7 lines 4-7 + truncation R4, given the d sketches Y_n."""
    d = x.ndim
    ys = list(ys)
    qs = [thin_qr(y)[0] for y in ys]
    g = _core_slabwise(x, qs, chunk)
    us = [None] * d
    for n in range(d):
        r = int(ranks[n])
        if r < qs[n].shape[1]:
            us[n], _ = leading_left_singular_vectors(unfold(g, n), r)
    for n in range(d):
        if us[n] is not None:
            qs[n] = qs[n] @ us[n]
            g = ttm(g, us[n].T, n)
    err = tucker_error(x, g, qs, chunk) if with_error else None
    return qs, g, err, ys


def sthosvd(x: np.ndarray, om_steps: Sequence[Sequence[Optional[np.ndarray]]], ranks: Sequence[int],
            with_error: bool = True):
    """RSTHOSVD-KRP (Alg. 8) with per-step truncation (R4, R5, R6).

    G^(0) = X.  For i = 1..d (ascending):
      1. Y_i = G_(i) (Omega ⊙ ... without i) with step-i Omegas; for an already
         compressed mode j < i only the leading r_j rows of Omega_j are used (R5)
      2. Q = thin QR(Y_i)
      3. B = G ×_i Qᵀ
      4. U = leading r_i left singular vectors of B_(i) (Alg. 2 pattern)
      5. G <- B ×_i Uᵀ ; Q_i = Q U
    Returns (qs, core, err, ys) where ys[i] is the step-i sketch."""
    d = x.ndim
    g = x
    qs = []
    ys = []
    for i in range(d):
        om = []
        for j in range(d):
            if j == i:
                om.append(None)
            else:
                om.append(np.asarray(om_steps[i][j], dtype=np.float64)[: g.shape[j]])
        om[i] = np.ones((1, np.asarray(om_steps[i][(i + 1) % d]).shape[1]))  # placeholder, unused
        y = sketch_mode(g, om, i)
        ys.append(y)
        q, _ = thin_qr(y)
        b = ttm(g, q.T, i)
        r = int(ranks[i])
        if r < q.shape[1]:
            u, _ = leading_left_singular_vectors(unfold(b, i), r)
            q = q @ u
            b = ttm(b, u.T, i)
        g = b
        qs.append(q)
    err = tucker_error(x, g, qs) if with_error else None
    return qs, g, err, ys


# ----------------------------------------------------------------- NEXT-2: fresh-Ω KRP and dense-Gaussian variants
def rhosvd_fresh(x: np.ndarray, om_steps: Sequence[Sequence[Optional[np.ndarray]]], ranks: Sequence[int],
                 with_error: bool = True):
    """RHOSVD-KRP, Alg. 7 read literally: for every mode n a fresh sequence {Omega^(n)_j}_{j != n}
    (om_steps[n][j]) and Y_n = X_(n) (Omega^(n)_d ⊙ ... ⊙ Omega^(n)_1); then QR, core and truncation as in
    ``rhosvd``.  2dNR sketch flops instead of 4NR."""
    ys = [sketch_mode(x, om_steps[n], n) for n in range(x.ndim)]
    return _rhosvd_from_sketches(x, ys, ranks, None, with_error)


def rhosvd_gaussian(x: np.ndarray, om_dense: Sequence[np.ndarray], ranks: Sequence[int], with_error: bool = True):
    """RHOSVD with dense Gaussian test matrices (the paper's baseline, Table 1): Y_n = X_(n) Omega_n with
    Omega_n in R^{(N/I_n) x l} iid N(0,1), rows in the column order of X_(n)."""
    ys = [unfold(x, n) @ np.asarray(om_dense[n], dtype=np.float64) for n in range(x.ndim)]
    return _rhosvd_from_sketches(x, ys, ranks, None, with_error)


def sthosvd_gaussian(x: np.ndarray, om_dense: Sequence[np.ndarray], ranks: Sequence[int], with_error: bool = True):
    """RSTHOSVD with dense Gaussian test matrices (Table 1 baseline): step i sketches the current core,
    Y_i = G_(i) Omega_i with Omega_i in R^{(N_i/I_i) x l} (N_i = the current core size), then the
    Alg. 8 steps of ``sthosvd`` (QR, B = G ×_i Qᵀ, truncation by the SVD of B_(i))."""
    g = x
    qs = []
    for i in range(x.ndim):
        y = unfold(g, i) @ np.asarray(om_dense[i], dtype=np.float64)
        q, _ = thin_qr(y)
        b = ttm(g, q.T, i)
        r = int(ranks[i])
        if r < q.shape[1]:
            u, _ = leading_left_singular_vectors(unfold(b, i), r)
            q = q @ u
            b = ttm(b, u.T, i)
        g = b
        qs.append(q)
    err = tucker_error(x, g, qs) if with_error else None
    return qs, g, err


# ----------------------------------------------------------------- NEXT-4: Hadamard products of Tucker tensors (App. C)
def row_kron(a: np.ndarray, u: np.ndarray) -> np.ndarray:
    """Transposed Khatri-Rao product A ⊙ᵀ U = (Aᵀ ⊙ Uᵀ)ᵀ, the row-wise Kronecker product: row i is
    A(i,:) ⊗ U(i,:), column index a * s + alpha (U's index fastest)."""
    a = np.asarray(a, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    return (a[:, :, None] * u[:, None, :]).reshape(a.shape[0], -1)


def _tensor_kron(f: np.ndarray, g: np.ndarray) -> np.ndarray:
    """F ⊗ G with H(A, B, C) = F(a,b,c) G(alpha,beta,gamma), A = alpha + a * q (P:960-962, 0-based)."""
    h = np.multiply.outer(f, g)  # axes a, b, c, alpha, beta, gamma
    d = f.ndim
    perm = [x for k in range(d) for x in (k, d + k)]  # a, alpha, b, beta, c, gamma
    h = np.transpose(h, perm)
    return h.reshape([f.shape[k] * g.shape[k] for k in range(d)])


def hadamard_tucker_explicit(f, xs, g, ys) -> np.ndarray:
    """Z = X ∗ Y formed explicitly (small sizes only): X = F ×_n A_n, Y = G ×_n U_n."""
    return multi_ttm(np.asarray(f, dtype=np.float64), list(xs)) * multi_ttm(np.asarray(g, dtype=np.float64), list(ys))


def hadamard_tucker_rhosvd(f, xs, g, ys, ranks: Sequence[int], om: Sequence[Sequence[Optional[np.ndarray]]]):
    """Alg. 9 (randomized HOSVD of the Hadamard product of two 3-way Tucker tensors), step by step:
    1. Ω_{i,j} ∈ R^{n_j x l_i} (om[i][j], j != i; l_i = r_i + oversampling)
    2. for each mode i: the sketch Z_(i)(⊙_{j != i, descending} Ω_{i,j}) computed through the structure
       (P:989-993): M_j = (A_jᵀ ⊙ U_jᵀ) Ω_{i,j}  (q_j s_j x l_i), then
       T = (F ⊗ G)_(i) (M_k ⊙ M_j)  (k > j the other two modes), then  Ẑ_i = (A_i ⊙ᵀ U_i) T
       — the n_1 n_2 n_3 product Z is never formed;  Q_i = orth(Ẑ_i)
    3. H = (F ⊗ G) ×_i Q_iᵀ(A_i ⊙ᵀ U_i)  (line 10, reading R23: its X, Y, Z are the orthonormal Q_i)
    4. for r_i < l_i: truncation by the HOSVD of H (reading R4 applied to Alg. 9)
    Returns (qs, core)."""
    d = 3
    f = np.asarray(f, dtype=np.float64)
    g = np.asarray(g, dtype=np.float64)
    fg = _tensor_kron(f, g)
    qs = []
    for i in range(d):
        others = [j for j in range(d) if j != i]
        ms = {j: row_kron(xs[j], ys[j]).T @ np.asarray(om[i][j], dtype=np.float64) for j in others}
        # column-wise KR of the others in descending mode order: rows (j fastest, then k)
        kr = khatri_rao(ms[others[1]], ms[others[0]])
        t = unfold(fg, i) @ kr
        zhat = row_kron(xs[i], ys[i]) @ t
        qs.append(thin_qr(zhat)[0])
    h = fg
    for i in range(d):
        h = ttm(h, qs[i].T @ row_kron(xs[i], ys[i]), i)
    us = [None] * d
    for i in range(d):
        if int(ranks[i]) < qs[i].shape[1]:
            us[i], _ = leading_left_singular_vectors(unfold(h, i), int(ranks[i]))
    for i in range(d):
        if us[i] is not None:
            qs[i] = qs[i] @ us[i]
            h = ttm(h, us[i].T, i)
    return qs, h


# ----------------------------------------------------------------- deterministic baselines (context for NEXT-1)
def hosvd(x: np.ndarray, ranks: Sequence[int]):
    """Truncated HOSVD (the paper's deterministic baseline, Table 1 / Fig. 2): U_n = leading r_n left
    singular vectors of X_(n); G = X ×_1 U_1ᵀ ... ×_d U_dᵀ.  Returns (us, core, err)."""
    us = [leading_left_singular_vectors(unfold(x, n), int(r))[0] for n, r in enumerate(ranks)]
    g = multi_ttm(x, [u.T for u in us])
    return us, g, tucker_error(x, g, us)


def sthosvd_deterministic(x: np.ndarray, ranks: Sequence[int]):
    """Truncated STHOSVD (deterministic baseline): for i = 1..d, U_i = leading r_i left singular vectors of the
    current core's mode-i unfolding, G <- G ×_i U_iᵀ (the Alg. 8 pattern with the exact SVD in place of the
    sketch).  Returns (us, core, err)."""
    g = x
    us = []
    for i, r in enumerate(ranks):
        u, _ = leading_left_singular_vectors(unfold(g, i), int(r))
        us.append(u)
        g = ttm(g, u.T, i)
    return us, g, tucker_error(x, g, us)


# ----------------------------------------------------------------- accounting
def sketch_flops(dims: Sequence[int], R: int, all_modes: bool = True) -> int:
    """Algorithmic sketch flops: 4·N·R memoized all-modes (Table 1
    reading R8), 2·N·R for one mode."""
    N = int(np.prod(dims, dtype=np.int64))
    return (4 if all_modes else 2) * N * int(R)
