"""Pins for the fp64 oracle (host only, no GPU).

Each test checks the oracle against something other than itself: a worked
example printed in SPEC/derived by hand from the definition, brute force with
explicit Python loops, a closed form, a textbook special case, or an invariant
the paper states.  A plausible mistake in the oracle (a dropped term, a wrong
sign or index, transposed operands, the Def. 2.2 KR order instead of the
P:522 order) fails at least one of these.
"""
import itertools
import math

import numpy as np
import pytest

import oracle
import synth
from conftest import read_golden


def _rng(seed):
    return np.random.default_rng(seed)


def _rand_omegas(dims, R, seed):
    g = _rng(seed)
    return [g.standard_normal((n, R)) for n in dims]


# ----------------------------------------------------------------- tensor algebra
def test_unfold_worked_example():
    """2x2x2 data 1..8 (first-index-fastest), mode 2 -> [[1,2,5,6],[3,4,7,8]]."""
    g = read_golden("unfold_2x2x2.txt")
    dims = [int(v) for v in g[0]]
    x = oracle.as_tensor(np.array(g[1]), dims)
    mode = int(g[2][0]) - 1
    assert np.array_equal(oracle.unfold(x, mode), np.array(g[3:5]))


def test_unfold_column_map_bruteforce():
    """Column index of x[i] in X_(n) is sum_{k!=n} i_k J_k, J_k = prod_{m<k,m!=n} I_m."""
    dims = (3, 4, 2, 5)
    flat = np.arange(np.prod(dims), dtype=np.float64)
    x = oracle.as_tensor(flat, dims)
    for n in range(4):
        u = oracle.unfold(x, n)
        for idx in itertools.product(*[range(v) for v in dims]):
            col, J = 0, 1
            for k in range(4):
                if k == n:
                    continue
                col += idx[k] * J
                J *= dims[k]
            lin = sum(idx[k] * int(np.prod(dims[:k])) for k in range(4))
            assert u[idx[n], col] == lin
        assert np.array_equal(oracle.fold(u, n, dims), x)


def test_kron_block_definition():
    """P:83-84 block layout; compared against numpy's independent kron."""
    g = _rng(1)
    a, b = g.standard_normal((2, 3)), g.standard_normal((4, 2))
    assert np.allclose(oracle.kron(a, b), np.kron(a, b), rtol=0, atol=1e-15)
    assert np.array_equal(oracle.kron(np.array([[1.0, 2.0]]), np.array([[3.0, 4.0]])), [[3, 4, 6, 8]])


def test_khatri_rao_examples():
    """S:95-96 / S:179: [[1],[2]] ⊙ [[3],[4]] = [3,4,6,8]^T ; ones(1,r) ⊙ B = B."""
    assert np.array_equal(oracle.khatri_rao(np.array([[1.0], [2.0]]), np.array([[3.0], [4.0]])),
                          [[3], [4], [6], [8]])
    b = _rng(2).standard_normal((5, 3))
    assert np.array_equal(oracle.khatri_rao(np.ones((1, 3)), b), b)


def test_mixed_product_property():
    """(A ⊗ B)(C ⊙ D) = (AC) ⊙ (BD) — pins KR row order against kron."""
    g = _rng(3)
    A, B = g.standard_normal((2, 3)), g.standard_normal((4, 5))
    C, D = g.standard_normal((3, 6)), g.standard_normal((5, 6))
    lhs = oracle.kron(A, B) @ oracle.khatri_rao(C, D)
    rhs = oracle.khatri_rao(A @ C, B @ D)
    assert np.allclose(lhs, rhs, rtol=1e-13, atol=1e-13)


# ----------------------------------------------------------------- the sketch
def _bruteforce_sketch(x, omegas, n):
    """Column identity Y_n(:,j) = X ×_{k!=n} ω_k^(j)ᵀ written as explicit loops."""
    dims = x.shape
    R = omegas[(n + 1) % len(dims)].shape[1]
    y = np.zeros((dims[n], R))
    for idx in itertools.product(*[range(v) for v in dims]):
        for j in range(R):
            w = 1.0
            for k, ik in enumerate(idx):
                if k != n:
                    w *= omegas[k][ik, j]
            y[idx[n], j] += x[idx] * w
    return y


@pytest.mark.parametrize("dims", [(3, 4, 5), (2, 3, 4, 5), (2, 3, 2, 3, 2), (4, 3)])
def test_sketch_bruteforce(dims):
    """BASELINE north_star pin (1): brute force on tiny tensors, every mode."""
    g = _rng(sum(dims))
    x = g.standard_normal(dims)
    om = _rand_omegas(dims, 3, 7)
    for n in range(len(dims)):
        ref = _bruteforce_sketch(x, om, n)
        got = oracle.sketch_mode(x, om, n)
        assert np.allclose(got, ref, rtol=1e-12, atol=1e-12), n


def test_sketch_definition_order_matters():
    """The Def. 2.2 order (Omega_1 ⊙ ... ⊙ Omega_d) does NOT pair with the unfolding;
    the P:522 order does (reading R1) — guards against swapping the KR order."""
    dims = (2, 3, 4)
    x = _rng(5).standard_normal(dims)
    om = _rand_omegas(dims, 2, 6)
    wrong = oracle.unfold(x, 0) @ oracle.khatri_rao(om[1], om[2])
    right = oracle.unfold(x, 0) @ oracle.khatri_rao(om[2], om[1])
    assert np.allclose(oracle.sketch_mode(x, om, 0), right)
    assert not np.allclose(wrong, right)


def test_sketch_integer_worked_example():
    """Hand-derived integer example (tests/golden/krp_int_2x2x2.txt); exact."""
    g = read_golden("krp_int_2x2x2.txt")
    x = oracle.as_tensor(np.arange(1, 9, dtype=np.float64), (2, 2, 2))
    om = [np.array([[1.0, -1.0], [2.0, 0.0]]), np.array([[0.0, 1.0], [1.0, 2.0]]),
          np.array([[1.0, 1.0], [-1.0, 3.0]])]
    for blk in range(3):
        n = int(g[3 * blk][0]) - 1
        expect = np.array(g[3 * blk + 1:3 * blk + 3])
        assert np.array_equal(oracle.sketch_mode(x, om, n), expect), n


@pytest.mark.parametrize("d", [3, 4, 5])
def test_rank_one_closed_form(d):
    """BASELINE north_star pin (2): X = a∘b∘c => Y_1 = a·((bᵀΩ_2)∘(cᵀΩ_3)) columnwise (d = 3, 4, 5)."""
    g = _rng(10 + d)
    dims = (5, 4, 3, 2, 3)[:d]
    vecs = [g.standard_normal(n) for n in dims]
    x = vecs[0]
    for v in vecs[1:]:
        x = np.multiply.outer(x, v)
    om = _rand_omegas(dims, 4, 11)
    for n in range(d):
        prod = np.ones(4)
        for k in range(d):
            if k != n:
                prod = prod * (vecs[k] @ om[k])
        assert np.allclose(oracle.sketch_mode(x, om, n), np.outer(vecs[n], prod), rtol=1e-12, atol=1e-12)


def test_d2_textbook_gemm():
    """d=2: Y_1 = X Ω_2 and Y_2 = Xᵀ Ω_1."""
    g = _rng(20)
    x = g.standard_normal((6, 7))
    om = _rand_omegas((6, 7), 3, 21)
    assert np.allclose(oracle.sketch_mode(x, om, 0), x @ om[1], rtol=1e-13, atol=1e-13)
    assert np.allclose(oracle.sketch_mode(x, om, 1), x.T @ om[0], rtol=1e-13, atol=1e-13)


def test_fiber_sums():
    """Single-column all-ones factors give the mode-n fiber sums."""
    dims = (3, 4, 5)
    x = _rng(22).standard_normal(dims)
    om = [np.ones((n, 1)) for n in dims]
    for n in range(3):
        axes = tuple(k for k in range(3) if k != n)
        assert np.allclose(oracle.sketch_mode(x, om, n)[:, 0], x.sum(axis=axes), rtol=1e-13, atol=1e-13)


def test_linearity_and_mode_permutation():
    dims = (3, 4, 5)
    g = _rng(23)
    x1, x2 = g.standard_normal(dims), g.standard_normal(dims)
    om = _rand_omegas(dims, 3, 24)
    for n in range(3):
        lhs = oracle.sketch_mode(2.0 * x1 - 3.0 * x2, om, n)
        rhs = 2.0 * oracle.sketch_mode(x1, om, n) - 3.0 * oracle.sketch_mode(x2, om, n)
        assert np.allclose(lhs, rhs, rtol=1e-12, atol=1e-12)
    perm = (2, 0, 1)
    xp = np.transpose(x1, perm)
    omp = [om[p] for p in perm]
    for n in range(3):
        assert np.allclose(oracle.sketch_mode(xp, omp, n), oracle.sketch_mode(x1, om, perm[n]), rtol=1e-12)


def test_chunked_and_rows_match_unchunked():
    cfg = synth.config("c1")
    x = synth.tensor(cfg, 3)
    om = synth.omegas(cfg.dims, cfg.R, 3)
    X = oracle.as_tensor(x, cfg.dims)
    for n in range(3):
        a = oracle.sketch_mode(X, om, n)
        b = oracle.sketch_mode(X, om, n, chunk=5)
        assert np.allclose(a, b, rtol=1e-12, atol=1e-10)
        rows = [0, 17, 63]
        assert np.allclose(oracle.sketch_mode_rows(x, cfg.dims, om, n, rows), a[rows], rtol=1e-12, atol=1e-10)


def test_isotropy_expected_energy():
    """Lemma 2.3: KRP columns are isotropic, so E_Ω ||Y_n||_F^2 = R ||X||_F^2."""
    dims = (4, 5, 6)
    x = _rng(30).standard_normal(dims)
    R, draws = 4, 600
    nx2 = float(np.sum(x * x))
    ratios = []
    for t in range(draws):
        om = _rand_omegas(dims, R, 1000 + t)
        ratios.append(np.sum(oracle.sketch_mode(x, om, 1) ** 2) / (R * nx2))
    m, s = np.mean(ratios), np.std(ratios) / math.sqrt(draws)
    assert abs(m - 1.0) < 4 * s, (m, s)


def test_sketch_flops_accounting():
    """4NR all modes memoized, 2NR per mode."""
    assert oracle.sketch_flops((64, 64, 64), 10) == 4 * 64 ** 3 * 10
    assert oracle.sketch_flops((64, 64, 64), 10, all_modes=False) == 2 * 64 ** 3 * 10


# ----------------------------------------------------------------- QR, TTM
def _gram_schmidt(y):
    """Classical Gram-Schmidt with reorthogonalisation, explicit loops (independent QR)."""
    m, r = y.shape
    q = np.zeros((m, r))
    rr = np.zeros((r, r))
    for j in range(r):
        v = y[:, j].copy()
        for _ in range(2):
            for i in range(j):
                c = q[:, i] @ v
                rr[i, j] += c
                v -= c * q[:, i]
        rr[j, j] = np.linalg.norm(v)
        q[:, j] = v / rr[j, j]
    return q, rr


def test_thin_qr_properties_and_uniqueness():
    y = _rng(40).standard_normal((30, 6))
    q, r = oracle.thin_qr(y)
    assert np.allclose(q.T @ q, np.eye(6), atol=1e-13)
    assert np.allclose(q @ r, y, atol=1e-12)
    assert np.all(np.diag(r) > 0) and np.allclose(np.tril(r, -1), 0)
    q2, r2 = _gram_schmidt(y)
    assert np.allclose(q, q2, atol=1e-11) and np.allclose(r, r2, atol=1e-11)


def test_ttm_definition_loops():
    """Y = X ×_n A: y[..i_n'..] = sum_{i_n} a[i_n', i_n] x[..i_n..], explicit loops."""
    dims = (3, 4, 2)
    x = _rng(41).standard_normal(dims)
    a = _rng(42).standard_normal((5, 4))
    y = oracle.ttm(x, a, 1)
    ref = np.zeros((3, 5, 2))
    for i, j, k, l in itertools.product(range(3), range(5), range(2), range(4)):
        ref[i, j, k] += a[j, l] * x[i, l, k]
    assert np.allclose(y, ref, atol=1e-13)


def test_multi_ttm_identity_and_norm():
    dims = (4, 5, 6)
    x = _rng(43).standard_normal(dims)
    assert np.allclose(oracle.multi_ttm(x, [np.eye(n) for n in dims]), x)
    qs = [np.linalg.qr(_rng(44 + k).standard_normal((n, 2)))[0].T for k, n in enumerate(dims)]
    g = oracle.multi_ttm(x, qs)
    assert np.linalg.norm(g) <= np.linalg.norm(x) + 1e-12
    # order of application does not matter (multilinearity)
    y = x
    for n in (2, 0, 1):
        y = oracle.ttm(y, qs[n], n)
    assert np.allclose(y, g, rtol=1e-13, atol=1e-13)


# ----------------------------------------------------------------- Tucker algorithms
def _noise_free_tucker(dims, core_dims, seed):
    cfg = synth.Config("t", tuple(dims), 0, tuple(core_dims), "tucker", core=tuple(core_dims))
    return oracle.as_tensor(synth.tensor_slab(cfg, seed, 0, dims[-1]).astype(np.float64), dims), cfg


def _noise_free_tucker64(dims, core_dims, seed):
    """fp64 (not rounded to fp32) noise-free Tucker tensor, for exact-recovery pins."""
    cfg = synth.Config("t", tuple(dims), 0, tuple(core_dims), "tucker", core=tuple(core_dims))
    core, us, _ = synth.tucker_parts(cfg, seed)
    return oracle.multi_ttm(core, us)


@pytest.mark.parametrize("dims,core,R,ranks", [((20, 18, 16), (3, 4, 2), 6, (3, 4, 2)),
                                               ((15, 15, 15), (2, 3, 2), 5, (5, 5, 5)),
                                               ((10, 9, 8, 7), (2, 2, 3, 2), 4, (2, 2, 3, 2))])
def test_rhosvd_exact_recovery(dims, core, R, ranks):
    """North-star pin (3): noise-free Tucker with ranks <= targets -> rel. error < 1e-12."""
    x = _noise_free_tucker64(dims, core, 5)
    om = _rand_omegas(dims, R, 6)
    _, _, err, _ = oracle.rhosvd(x, om, ranks)
    assert err < 1e-12, err


def test_sthosvd_exact_recovery():
    dims, core, R = (12, 11, 10, 9), (2, 3, 2, 2), 5
    x = _noise_free_tucker64(dims, core, 8)
    oms = [[None if j == i else _rng(100 * i + j).standard_normal((n, R)) for j, n in enumerate(dims)]
           for i in range(4)]
    _, _, err, _ = oracle.sthosvd(x, oms, core)
    assert err < 1e-12, err


def _rand_tensor_with_decay(dims, seed):
    x = _rng(seed).standard_normal(dims)
    for n, v in enumerate(dims):
        shape = [1] * len(dims)
        shape[n] = v
        x = x * (0.6 ** np.arange(v)).reshape(shape)
    return x


def test_rhosvd_error_bounds():
    """Thm 5.1 proof step: ||X-X̂||² <= Σ_n ||(I-Q_nQ_nᵀ)X_(n)||²;
    Eckart-Young lower bound ||X-X̂||² >= max_n Σ_{j>r_n} σ_j²(X_(n)) (textbook);
    orthogonal projection: ||X-X̂||² = ||X||² - ||G||²."""
    dims, R, ranks = (14, 12, 10), 6, (4, 3, 5)
    x = _rand_tensor_with_decay(dims, 50)
    om = _rand_omegas(dims, R, 51)
    qs, g, err, _ = oracle.rhosvd(x, om, ranks)
    e2 = err ** 2 * np.sum(x * x)
    upper = sum(np.sum((oracle.unfold(x, n) - qs[n] @ (qs[n].T @ oracle.unfold(x, n))) ** 2) for n in range(3))
    lower = max(np.sum(np.linalg.svd(oracle.unfold(x, n), compute_uv=False)[ranks[n]:] ** 2) for n in range(3))
    assert lower <= e2 * (1 + 1e-12) <= upper * (1 + 1e-12)
    assert abs(e2 - (np.sum(x * x) - np.sum(g * g))) < 1e-10 * np.sum(x * x)
    for q, r in zip(qs, ranks):
        assert q.shape[1] == r and np.allclose(q.T @ q, np.eye(r), atol=1e-12)


def test_rhosvd_truncation_is_hosvd_of_the_core():
    """Reading R4 ("hosvd on the core"): every U_n = Qfull_nᵀ Q_n diagonalises the mode-n Gram of the
    UNTRUNCATED core G0 with its r_n largest eigenvalues (checked with a symmetric eigen-solver, not the
    oracle's SVD); a sequential (ST) truncation of the core fails this for the second truncated mode."""
    dims, R, ranks = (14, 12, 10), 6, (3, 4, 6)
    x = _rand_tensor_with_decay(dims, 52)
    om = _rand_omegas(dims, R, 53)
    qs, g, _, ys = oracle.rhosvd(x, om, ranks)
    qf = [oracle.thin_qr(y)[0] for y in ys]
    g0 = oracle.multi_ttm(x, [q.T for q in qf])
    for n, r in enumerate(ranks):
        if r == R:
            assert np.allclose(qs[n], qf[n], atol=1e-13)
            continue
        u = qf[n].T @ qs[n]
        h = oracle.unfold(g0, n) @ oracle.unfold(g0, n).T
        ev = np.linalg.eigvalsh(h)[::-1][:r]
        m = u.T @ h @ u
        assert np.allclose(np.diag(m), ev, rtol=1e-10, atol=1e-12 * ev[0])
        assert np.abs(m - np.diag(np.diag(m))).max() < 1e-10 * ev[0]
    assert np.allclose(g, oracle.multi_ttm(g0, [(qf[n].T @ qs[n]).T for n in range(3)]), atol=1e-12)


def test_ranks_equal_dims_exact():
    """ranks = dims (sketch width = every mode size) -> exact reconstruction."""
    dims = (5, 5, 5)
    x = _rng(60).standard_normal(dims)
    om = _rand_omegas(dims, 5, 61)
    _, _, err, _ = oracle.rhosvd(x, om, (5, 5, 5))
    assert err < 1e-12


def test_sthosvd_error_identity_and_bound():
    """Thm 5.2 proof: ||X-X̂||² = Σ_i ||X̂^(i-1) - X̂^(i)||²
    and <= Σ_i ||(I-Q_iQ_iᵀ) G^(i-1)_(i)||² (here with the truncated Q_i, which are
    orthonormal, so each term is the projection residual of that step)."""
    dims, R, ranks = (10, 9, 8, 7), 5, (3, 4, 3, 2)
    x = _rand_tensor_with_decay(dims, 90)
    oms = [[None if j == i else _rng(200 + 10 * i + j).standard_normal((n, R)) for j, n in enumerate(dims)]
           for i in range(4)]
    qs, g, err, _ = oracle.sthosvd(x, oms, ranks)
    e2 = err ** 2 * np.sum(x * x)
    # partial reconstructions X̂^(i) = G^(i) ×_{j<=i} Q_j (with G^(i) the core after step i)
    gi = x
    prev = x
    parts, resid = 0.0, 0.0
    for i in range(4):
        gu = oracle.unfold(gi, i)
        resid += np.sum((gu - qs[i] @ (qs[i].T @ gu)) ** 2)
        gi = oracle.ttm(gi, qs[i].T, i)
        xh = oracle.multi_ttm(gi, [qs[j] if j <= i else None for j in range(4)])
        parts += np.sum((prev - xh) ** 2)
        prev = xh
    assert abs(parts - e2) < 1e-10 * np.sum(x * x)
    assert e2 <= resid * (1 + 1e-12)
    assert np.allclose(gi, g, atol=1e-12)


# ----------------------------------------------------------------- multi-GPU host identity
def test_slab_sum_identity():
    """Sharding along the last mode: the sketches of modes n<d are sums of
    per-slab sketches; the rows of Y_d are the per-slab Y_d rows."""
    cfg = synth.config("c1").scaled((8, 6, 12))
    x = synth.tensor(cfg, 4)
    om = synth.omegas(cfg.dims, 5, 4)
    X = oracle.as_tensor(x, cfg.dims)
    full = oracle.sketch_all_modes(X, om)
    G = 3
    parts = []
    for g_ in range(G):
        k0, k1 = 4 * g_, 4 * (g_ + 1)
        slab = synth.tensor_slab(cfg, 4, k0, k1)
        assert np.array_equal(slab, x[k0 * 48:k1 * 48])  # generator is slab-consistent
        om_s = om[:2] + [om[2][k0:k1]]
        parts.append(oracle.sketch_all_modes(oracle.as_tensor(slab, (8, 6, 4)), om_s))
    for n in range(2):
        assert np.allclose(sum(p[n] for p in parts), full[n], rtol=1e-12, atol=1e-12)
    assert np.allclose(np.concatenate([p[2] for p in parts]), full[2], rtol=1e-12, atol=1e-12)


def test_synth_generator_recipe():
    """Generator sanity: orthonormal factors, noise level, smooth-function values (0-based)."""
    cfg = synth.config("c1")
    core, us, nrm = synth.tucker_parts(cfg, 0)
    for u in us:
        assert np.allclose(u.T @ u, np.eye(u.shape[1]), atol=1e-13)
    x = synth.tensor(cfg, 0).astype(np.float64)
    x0 = oracle.multi_ttm(core, us).reshape(-1, order="F")
    rel = np.linalg.norm(x - x0) / np.linalg.norm(x0)
    assert 0.9e-4 < rel < 1.1e-4
    c5 = synth.config("c5").scaled((8, 8, 4))
    v = synth.tensor_slab(dataclasses_replace_eta0(c5), 0, 0, 4)
    assert v[0] == 1.0
    assert np.isclose(v[1 + 8 * 2 + 64 * 3], 1.0 / (1 + 1 / 8 + 2 / 8 + 3 / 4), rtol=1e-7)


def dataclasses_replace_eta0(cfg):
    import dataclasses
    return dataclasses.replace(cfg, eta=0.0)


@pytest.mark.parametrize("dims", [(5, 4, 3), (3, 4, 2, 5), (2, 3, 2, 3, 2), (7, 2)])
def test_sampled_rows_ttv_matches_explicit_kr(dims):
    """The full-size sampled-row oracle (column identity, multi-TTV) against the explicit-KR sketch,
    every row of every mode, on random tensors (pins sketch_rows_ttv)."""
    g = _rng(11)
    flat = g.standard_normal(int(np.prod(dims)))
    om = _rand_omegas(dims, 3, 12)
    x = oracle.as_tensor(flat, dims)
    for n in range(len(dims)):
        ref = oracle.sketch_mode(x, om, n)
        got = oracle.sketch_rows_ttv(flat, dims, om, n, list(range(dims[n])))
        assert np.allclose(got, ref, rtol=1e-12, atol=1e-12), n


def test_chunked_rhosvd_and_error_match_unchunked():
    """Memory-only chunking (last-mode slabs) changes the fp64 summation order, never the terms: the chunked
    sketch, core and Tucker error of rhosvd equal the unchunked ones to rounding (pins the chunked branches
    of sketch_mode, _core_slabwise and tucker_error that the full-size GPU tests use)."""
    cfg = synth.config("c2").scaled((24, 20, 18))
    x = oracle.as_tensor(synth.tensor(cfg, 4), cfg.dims)
    om = synth.omegas(cfg.dims, cfg.R if cfg.R <= 18 else 12, 4)
    ranks = (5, 5, 5)
    q0, g0, e0, y0 = oracle.rhosvd(x, om, ranks, chunk=None)
    for chunk in (1, 5, 7, 17):
        q1, g1, e1, y1 = oracle.rhosvd(x, om, ranks, chunk=chunk)
        for a, b in zip(y0, y1):
            assert np.allclose(a, b, rtol=1e-12, atol=1e-12 * np.abs(a).max())
        assert abs(e1 - e0) <= 1e-12
        assert np.allclose(np.abs(g1), np.abs(g0), rtol=1e-9, atol=1e-12)
        # the chunked error of the same decomposition equals the unchunked one
        assert abs(oracle.tucker_error(x, g0, q0, chunk=chunk) - e0) <= 1e-13


def test_deterministic_hosvd_sthosvd_bounds():
    """HOSVD / STHOSVD baselines (context for the Cauchy workload, NEXT-1): the textbook bounds
    ||X - X̂||² <= Σ_n Σ_{j>r_n} σ_j²(X_(n)) (De Lathauwer et al. 2000; P:612 tail sums) and >= the largest
    single-mode tail (Eckart–Young), exact recovery when the ranks cover the multilinear rank, and the
    paper's observation that the randomized KRP variants come close to HOSVD on the Cauchy tensor."""
    cfg = synth.config("cauchy").scaled((14, 12, 10, 9))
    x = oracle.as_tensor(synth.tensor(cfg, 0), cfg.dims)
    ranks = (4, 4, 4, 4)
    tails = [float(np.sum(np.linalg.svd(oracle.unfold(x, n), compute_uv=False)[r:] ** 2)) for n, r in enumerate(ranks)]
    nx2 = float(np.sum(x ** 2))
    for fn in (oracle.hosvd, oracle.sthosvd_deterministic):
        us, g, err = fn(x, ranks)
        e2 = err ** 2 * nx2
        assert e2 <= sum(tails) * (1 + 1e-9) and e2 >= max(tails) * (1 - 1e-9)
        for u, r in zip(us, ranks):
            assert np.allclose(u.T @ u, np.eye(r), atol=1e-12)
    # exact recovery of a multilinear-rank-(2,2,2) tensor
    g0 = _rng(77).standard_normal((2, 2, 2))
    fac = [np.linalg.qr(_rng(78 + k).standard_normal((n, 2)))[0] for k, n in enumerate((7, 6, 5))]
    xt = oracle.multi_ttm(g0, fac)
    assert oracle.hosvd(xt, (2, 2, 2))[2] < 1e-12 and oracle.sthosvd_deterministic(xt, (2, 2, 2))[2] < 1e-12
    # the memoized randomized variant with no oversampling is within a small factor of HOSVD (Fig. 2 setup)
    om = synth.omegas(cfg.dims, 4, 3)
    e_memo = oracle.rhosvd(x, om, ranks)[2]
    assert oracle.hosvd(x, ranks)[2] <= e_memo <= 10 * oracle.hosvd(x, ranks)[2]


def test_fresh_and_gaussian_variants_reduce_to_memo():
    """NEXT-2 pins.  (1) Alg. 7 with every mode's fresh sequence equal to the memoized set IS RHOSVD-KRP-MEMO
    (P:571).  (2) A dense test matrix equal to the Khatri-Rao product turns the Gaussian sketch into the KRP
    sketch, which pins the dense variant's unfolding / row order.  (3) Fresh sequences and
    dense Gaussians both recover a noise-free Tucker tensor exactly (the randomized range finder)."""
    cfg = synth.config("c2").scaled((12, 10, 9))
    x = oracle.as_tensor(synth.tensor(cfg, 2), cfg.dims)
    R, ranks = 6, (4, 4, 4)
    om = synth.omegas(cfg.dims, R, 2)
    q0, g0, e0, y0 = oracle.rhosvd(x, om, ranks)
    same = [[None if j == n else om[j] for j in range(3)] for n in range(3)]
    q1, g1, e1, y1 = oracle.rhosvd_fresh(x, same, ranks)
    assert abs(e1 - e0) < 1e-13 and all(np.allclose(a, b, rtol=1e-13, atol=1e-13) for a, b in zip(y0, y1))
    dense = [oracle.kr_for_mode(om, n) for n in range(3)]
    q2, g2, e2, y2 = oracle.rhosvd(x, om, ranks)
    _, _, e3, _ = oracle.rhosvd_gaussian(x, dense, ranks)
    assert abs(e3 - e0) < 1e-12
    for n in range(3):
        assert np.allclose(oracle.unfold(x, n) @ dense[n], y0[n], rtol=1e-12, atol=1e-12)
    # exact recovery with genuinely fresh / dense randomness
    ct = synth.Config("t", (12, 10, 9), 6, (3, 3, 3), "tucker", core=(3, 3, 3))
    core, us, _ = synth.tucker_parts(ct, 1)
    xt = oracle.multi_ttm(core, us)  # fp64, exactly multilinear rank (3, 3, 3)
    assert oracle.rhosvd_fresh(xt, synth.rhosvd_fresh_omegas(ct.dims, 6, 1), (3, 3, 3))[2] < 1e-12
    assert oracle.rhosvd_gaussian(xt, synth.dense_gaussian(ct.dims, 6, 1), (3, 3, 3))[2] < 1e-12
    assert oracle.sthosvd_gaussian(xt, synth.dense_gaussian_sthosvd(ct.dims, (3, 3, 3), 6, 1), (3, 3, 3))[2] < 1e-12


def test_hadamard_tucker_structured_equals_explicit():
    """NEXT-4 pins (App. C): (1) the Hadamard product identity X ∗ Y = (F⊗G) ×_n (A_n ⊙ᵀ U_n) (eq. (C.1),
    Kressner–Periša Lemma 3.1) holds elementwise; (2) Alg. 9's structured sketch equals the explicit MTTKRP of Z
    with the same Ω (the derivation at P:989-993); (3) its core equals Z ×_n Q_nᵀ, so Ẑ is the orthogonal
    projection of Z; (4) with l_i >= q_i s_i (the multilinear rank of Z) the recompression is exact."""
    ns, qs_, ss = (9, 8, 7), (2, 3, 2), (3, 2, 3)
    f, xs, g, ys = synth.hadamard_tucker_inputs(ns, qs_, ss, 3)
    z = oracle.hadamard_tucker_explicit(f, xs, g, ys)
    # (1) elementwise identity through the row-wise Kronecker factors
    z2 = oracle.multi_ttm(_tk(f, g), [oracle.row_kron(a, u) for a, u in zip(xs, ys)])
    assert np.allclose(z, z2, rtol=1e-12, atol=1e-13)
    ls = (5, 4, 6)
    om = synth.hadamard_omegas(ns, ls, 3)
    qs, h = oracle.hadamard_tucker_rhosvd(f, xs, g, ys, ls, om)
    for i in range(3):
        omi = [np.ones((1, ls[i])) if j == i else om[i][j] for j in range(3)]
        y = oracle.sketch_mode(z, omi, i)
        q, _ = oracle.thin_qr(y)
        assert np.allclose(np.abs(q.T @ qs[i]), np.eye(ls[i]), atol=1e-8)  # same range, same Q up to signs
    assert np.allclose(h, oracle.multi_ttm(z, [q.T for q in qs]), rtol=1e-10, atol=1e-12)
    # (4) exact when every l_i covers q_i s_i
    lx = tuple(q * s for q, s in zip(qs_, ss))
    qx, hx = oracle.hadamard_tucker_rhosvd(f, xs, g, ys, lx, synth.hadamard_omegas(ns, lx, 4))
    assert oracle.tucker_error(z, hx, qx) < 1e-12


def _tk(f, g):
    from oracle.krp_oracle import _tensor_kron
    return _tensor_kron(np.asarray(f, dtype=np.float64), np.asarray(g, dtype=np.float64))


def test_leading_singular_vectors_canonical_signs():
    """Reading R24: U is LAPACK's left singular basis with each column's largest-magnitude entry made
    positive.  Pins: the columns are the singular vectors (M M^T u = s^2 u against the eigen-decomposition
    of M M^T), the sign rule holds, and flipping the input's sign pattern does not change U."""
    m = np.random.default_rng(3).standard_normal((12, 40)) * np.logspace(0, -3, 12)[:, None]
    u, s = oracle.leading_left_singular_vectors(m, 5)
    g = m @ m.T
    assert np.allclose(g @ u, u * s[:5] ** 2, rtol=1e-10, atol=1e-12 * s[0] ** 2)
    w, v = np.linalg.eigh(g)
    assert np.allclose(np.abs(u.T @ v[:, ::-1][:, :5]), np.eye(5), atol=1e-10)
    for t in range(5):
        i = int(np.argmax(np.abs(u[:, t])))
        assert u[i, t] > 0
    # any sign pattern LAPACK returns maps to the same canonical U
    flip = oracle.canonical_signs(-u)
    assert np.array_equal(flip, u)
