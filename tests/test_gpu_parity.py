"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded inputs.

Every sketch runs on the tcgen05 3xTF32 kernels (the library has no other backend).  Tolerances
(BASELINE north_star): per-mode relative Frobenius error of Y_n <= 1e-5; Tucker relative error within
1e-4 (absolute difference, reading R12).  Small-integer inputs are exact in 3xTF32 (hi = x, lo = 0) and
every partial sum stays below 2^24, so those cases are compared bit for bit (torch.equal).
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

Y_TOL = 1e-5
ERR_TOL = 1e-4
QTQ_TOL = 1e-6


@pytest.fixture(scope="module")
def krp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2507_23207_b200 as krp
    from paper_2507_23207_b200 import build
    build.build()
    yield krp


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _int_inputs(dims, R, seed):
    """X in {-3..3}, Ω in {-2..2}: tf32-exact values whose partial sums are integers below 2^24."""
    g = np.random.default_rng([seed, 4242])
    x = g.integers(-3, 4, int(np.prod(dims))).astype(np.float32)
    om = [g.integers(-2, 3, (n, R)).astype(np.float32) for n in dims]
    # bound on any partial sum: max |x| * max |Π_{k != n} Ω_k| * (N / I_n terms) < 2^24
    terms = int(np.prod(dims)) // min(dims)
    assert 3 * 2 ** (len(dims) - 1) * terms < 2 ** 24
    return x, om


# ----------------------------------------------------------------- the sketch
def test_integer_worked_example_bit_exact(krp):
    """Hand-derived example (tests/golden/krp_int_2x2x2.txt): exact on the device."""
    x = np.arange(1, 9, dtype=np.float32)
    om = [np.array([[1, -1], [2, 0]], np.float32), np.array([[0, 1], [1, 2]], np.float32),
          np.array([[1, 1], [-1, 3]], np.float32)]
    ref = oracle.sketch_all_modes(oracle.as_tensor(x, (2, 2, 2)), om)
    Y = krp.krp_sketch_all_modes(_dev(x), (2, 2, 2), [_dev(o) for o in om])
    for n in range(3):
        assert torch.equal(Y[n].cpu(), torch.from_numpy(ref[n].astype(np.float32))), n


# tcgen05-tiled shapes with ragged blocks: d = 3, 4, 5, and R > 64 (two column groups); R = 60 / 56 take the
# QH plan (Q's A_hi in TMEM, register accumulators), the c5 plan
INT_SHAPES = [((256, 200, 12), 24), ((96, 64, 40, 10), 16), ((16, 12, 10, 8, 6), 8), ((128, 96, 20), 100),
              ((384, 130, 3), 40), ((256, 192, 10), 60), ((200, 130, 6), 56), ((64, 40, 36, 5), 60)]


@pytest.mark.parametrize("dims,R", INT_SHAPES)
def test_integer_sketch_bit_exact_tcgen05(krp, dims, R):
    x, om = _int_inputs(dims, R, len(dims) * 1000 + R)
    ref = oracle.sketch_all_modes(oracle.as_tensor(x, dims), om)
    Y = krp.krp_sketch_all_modes(_dev(x), dims, [_dev(o) for o in om])
    for n in range(len(dims)):
        r32 = ref[n].astype(np.float32)
        assert np.array_equal(r32.astype(np.float64), ref[n]), "reference not exact in fp32"
        assert torch.equal(Y[n].cpu(), torch.from_numpy(r32)), (n, float((Y[n].cpu() - torch.from_numpy(r32)).abs().max()))


@pytest.mark.parametrize("dims,R", [((256, 200, 12), 24), ((96, 64, 40, 10), 16)])
def test_integer_single_mode_bit_exact(krp, dims, R):
    x, om = _int_inputs(dims, R, 77 + R)
    X = oracle.as_tensor(x, dims)
    for n in range(len(dims)):
        ref = oracle.sketch_mode(X, om, n).astype(np.float32)
        omn = [None if k == n else _dev(o) for k, o in enumerate(om)]
        Y = krp.krp_sketch_mode(_dev(x), dims, n, omn)
        assert torch.equal(Y.cpu(), torch.from_numpy(ref)), n


SHAPES = [
    ((3, 4, 5), 3), ((2, 3, 4, 5), 4), ((17, 33, 9), 7), ((64, 64, 64), 10), ((130, 7, 64), 5),
    ((256, 129, 3), 16), ((128, 128, 40), 40), ((256, 256, 17), 40), ((384, 128, 9), 64),
    ((16, 16, 16, 16, 16), 20), ((64, 64, 8, 8), 20), ((6, 5, 4, 3, 2, 2), 6), ((1000, 3), 2),
    ((128, 256, 7), 128), ((512, 128, 5), 30), ((200, 150, 6), 256), ((96, 80, 11), 65),
    ((384, 256, 9), 60), ((130, 260, 5), 52), ((300, 200, 4), 120),
    # every mode odd: no grouping has a 16-byte row pitch (the repack path)
    ((5, 7, 9), 4), ((33, 35, 37), 12),
    # degenerate cases: R = 1, unit modes (first, middle, last), a single-element tensor, d = 2
    ((128, 128, 128), 1), ((1, 128, 256), 8), ((128, 1, 256), 8), ((256, 128, 1), 8), ((1, 1, 1), 1),
    ((300, 260), 33), ((1, 7), 1),
    # the largest order the boundary accepts (d = 8, krp.h) and d = 7
    ((4, 3, 2, 3, 2, 2, 3), 5), ((3, 2, 4, 2, 3, 2, 2, 5), 6), ((130, 2, 2, 2, 2, 2, 2, 2), 9),
]


@pytest.mark.parametrize("dims,R", SHAPES)
def test_sketch_all_modes_random(krp, dims, R):
    x = synth.random_tensor(dims, seed=1, tag=len(dims))
    om = synth.omegas(dims, R, seed=2)
    ref = oracle.sketch_all_modes(oracle.as_tensor(x, dims), om)
    Y = krp.krp_sketch_all_modes(_dev(x), dims, [_dev(o) for o in om])
    for n in range(len(dims)):
        e = rel(Y[n].cpu().numpy(), ref[n])
        assert e <= Y_TOL, (n, e)


def test_sketch_misaligned_input(krp):
    """X at a 4-byte (not 16-byte) offset: TMA needs a 16-byte base, so the library stages the input."""
    dims, R = (64, 48, 20), 12
    x = synth.random_tensor(dims, seed=5, tag=3)
    om = synth.omegas(dims, R, seed=6)
    ref = oracle.sketch_all_modes(oracle.as_tensor(x, dims), om)
    buf = torch.zeros(x.size + 1, dtype=torch.float32, device="cuda")
    buf[1:].copy_(torch.from_numpy(x))
    Xv = buf[1:]
    assert Xv.data_ptr() % 16 != 0
    Y = krp.krp_sketch_all_modes(Xv, dims, [_dev(o) for o in om])
    for n in range(3):
        assert rel(Y[n].cpu().numpy(), ref[n]) <= Y_TOL


@pytest.mark.parametrize("dims,R", [((3, 4, 5), 3), ((128, 128, 128), 30), ((20, 128, 128, 8), 30),
                                    ((20, 20, 128, 128), 30), ((20, 20, 20, 128), 30), ((256, 64, 64), 17),
                                    ((64, 48, 40), 80)])
def test_sketch_single_mode(krp, dims, R):
    x = synth.random_tensor(dims, seed=3, tag=len(dims))
    om = synth.omegas(dims, R, seed=4)
    X = oracle.as_tensor(x, dims)
    for n in range(len(dims)):
        ref = oracle.sketch_mode(X, om, n)
        omn = [None if k == n else _dev(o) for k, o in enumerate(om)]
        Y = krp.krp_sketch_mode(_dev(x), dims, n, omn)
        e = rel(Y.cpu().numpy(), ref)
        assert e <= Y_TOL, (n, e)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_sketch_config_recipes_scaled(krp, name):
    """Each BASELINE config's recipe (value distribution, R) on dims the oracle finishes in seconds."""
    small = {"c1": (64, 64, 64), "c2": (256, 256, 128), "c3": (64, 64, 64, 32), "c4": (32, 32, 16, 16, 16),
             "c5": (512, 256, 64)}[name]
    cfg = synth.config(name).scaled(small)
    x = synth.tensor(cfg, 0)
    om = synth.omegas(cfg.dims, cfg.R, 0)
    ref = oracle.sketch_all_modes(oracle.as_tensor(x, cfg.dims), om)
    Y = krp.krp_sketch_all_modes(_dev(x), cfg.dims, [_dev(o) for o in om])
    for n in range(cfg.d):
        e = rel(Y[n].cpu().numpy(), ref[n])
        assert e <= Y_TOL, (n, e)


def test_sketch_host_buffers(krp):
    cfg = synth.config("c1")
    x = synth.tensor(cfg, 5)
    om = synth.omegas(cfg.dims, cfg.R, 5)
    ref = oracle.sketch_all_modes(oracle.as_tensor(x, cfg.dims), om)
    Xh = torch.from_numpy(x).pin_memory()
    Oh = [torch.from_numpy(o).pin_memory() for o in om]
    Y = krp.krp_sketch_all_modes_host(Xh, cfg.dims, Oh)
    for n in range(3):
        assert rel(Y[n].numpy(), ref[n]) <= Y_TOL


def test_sketch_is_deterministic(krp):
    dims, R = (256, 256, 64), 40
    x = _dev(synth.random_tensor(dims, 9))
    om = [_dev(o) for o in synth.omegas(dims, R, 9)]
    a = krp.krp_sketch_all_modes(x, dims, om)
    b = krp.krp_sketch_all_modes(x, dims, om)
    for u, v in zip(a, b):
        assert torch.equal(u, v)


@pytest.mark.parametrize("dims,R", [((256, 256, 64), 40), ((64, 32, 16, 8, 6), 20)])
def test_assembly_long_list_path(krp, dims, R, monkeypatch):
    """The assembly's two term-list paths (listed used slots / every (pair, slot) walked) give the same
    sums up to summation grouping (P(rho, r) = sum over col blocks and CTA slots)."""
    x = _dev(synth.random_tensor(dims, 13))
    om = [_dev(o) for o in synth.omegas(dims, R, 13)]
    a = krp.krp_sketch_all_modes(x, dims, om)
    monkeypatch.setenv("KRP_ASM_UNLISTED", "1")
    b = krp.krp_sketch_all_modes(x, dims, om)
    ref = oracle.sketch_all_modes(oracle.as_tensor(x.cpu().numpy(), dims), [o.cpu().numpy() for o in om])
    for n, (u, v) in enumerate(zip(a, b)):
        scale = float(np.abs(ref[n]).max())
        assert float((u - v).abs().max()) <= 1e-6 * scale, n
        assert float((v.double().cpu() - torch.from_numpy(ref[n])).abs().max()) <= 1e-5 * scale, n


# ----------------------------------------------------------------- the core contraction (mode-n product)
# Mode 0 with I_1 % 4 == 0 and J <= 64 runs on the tcgen05 3xTF32 kernel; the shapes below span several
# 128-column tiles with a ragged last tile, K chunks with a ragged tail (I_1 = 36, 100), J = 1 .. 64 and
# the N padding (J = 10, 30, 50); the other modes / I_1 % 4 != 0 take the fp32 FMA kernels.
TTM_CASES = [((128, 40, 33), 0, 30), ((36, 50, 7), 0, 1), ((100, 77, 5), 0, 50), ((64, 64, 64), 0, 64),
             ((32, 17, 3, 5), 0, 10), ((2048, 20, 9), 0, 60), ((30, 40, 20), 0, 20), ((40, 36, 20), 1, 30),
             ((24, 20, 36), 2, 12)]


@pytest.mark.parametrize("dims,n,J", TTM_CASES)
def test_ttm_vs_oracle(krp, dims, n, J):
    x = synth.random_tensor(dims, 31)
    a = np.random.default_rng([31, n, J]).standard_normal((J, dims[n])).astype(np.float32)
    y = krp.krp_ttm(_dev(x), dims, n, _dev(a)).cpu().numpy()
    out = list(dims)
    out[n] = J
    ref = oracle.ttm(oracle.as_tensor(x, dims), a, n)
    got = oracle.as_tensor(y, out)
    assert rel(got, ref) <= Y_TOL, rel(got, ref)
    # every element within a conservative 3xTF32 bound: per product the dropped lo*lo term and the tf32
    # rounding of the two lo operands (each < 2^-20 |a x| even for a truncating split), plus fp32
    # accumulation over I_n terms (gamma_I ~ I 2^-24), relative to its own scale sum_i |a_ji x_i|
    scale = oracle.ttm(np.abs(oracle.as_tensor(x, dims)), np.abs(a.astype(np.float64)), n)
    bound = (3 * 2.0 ** -20 + dims[n] * 2.0 ** -24) * scale
    assert np.all(np.abs(got - ref) <= bound + 1e-30)


def test_ttm_positive_data_has_bounded_rounding_bias(krp):
    """All-positive X and A (the c5 smooth tensor against its dominant factor column): rounding errors of one
    sign add coherently here.  Two sources are bounded by the kernel's design: a truncating tf32 split would
    drop ~3 2^-22 = 7e-7 relative (the kernel splits round-to-nearest), and the tensor core's accumulation
    into TMEM rounds toward zero (~0.6 ulp per accumulating MMA: 4.6e-6 low for K = 512 accumulated in
    TMEM), so accumulators hold one 32-wide K chunk (4 MMAs, ~1.4e-7) and chunks are summed in fp32
    round-to-nearest registers."""
    dims, J = (512, 300, 4), 16
    i, j, k = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in dims], indexing="ij")
    x = (1.0 / (1.0 + i / dims[0] + j / dims[1] + k / dims[2])).reshape(-1, order="F").astype(np.float32)
    a = np.random.default_rng(11).uniform(0.1, 1.0, (J, dims[0])).astype(np.float32)
    y = krp.krp_ttm(_dev(x), dims, 0, _dev(a)).cpu().numpy()
    ref = oracle.ttm(oracle.as_tensor(x, dims), a, 0)
    assert rel(oracle.as_tensor(y, (J,) + dims[1:]), ref) <= 3e-7


def test_ttm_tensor_core_is_exact_on_small_integers_and_deterministic(krp):
    """Small integers are tf32-exact (lo = 0) with integer partial sums < 2^24: bit-exact; and a repeat is
    bit-identical (fixed summation order)."""
    dims, J = (96, 300, 3), 40
    g = np.random.default_rng(5)
    x = g.integers(-3, 4, int(np.prod(dims))).astype(np.float32)
    a = g.integers(-2, 3, (J, dims[0])).astype(np.float32)
    y = krp.krp_ttm(_dev(x), dims, 0, _dev(a))
    ref = oracle.ttm(oracle.as_tensor(x, dims), a, 0)
    assert np.array_equal(oracle.as_tensor(y.cpu().numpy(), (J, 300, 3)), ref)
    xr = _dev(synth.random_tensor(dims, 6))
    ar = _dev(g.standard_normal((J, dims[0])))
    assert torch.equal(krp.krp_ttm(xr, dims, 0, ar), krp.krp_ttm(xr, dims, 0, ar))


# ----------------------------------------------------------------- rHOSVD / STHOSVD
def _check_factors(Q, ranks, tol=QTQ_TOL):
    for q, r in zip(Q, ranks):
        q = q.double().cpu().numpy()
        assert q.shape[1] == r
        dev = np.abs(q.T @ q - np.eye(r)).max()
        assert dev <= tol, dev


@pytest.mark.parametrize("name,small", [("c1", None), ("c2", (128, 128, 128)), ("c4", (32, 32, 24, 24, 24)),
                                        ("c5", (256, 256, 64)),
                                        # mode-0 TTM kernel with ragged i (100 % 32) and column (10500 % 256) tails
                                        ("c2", (100, 150, 70)),
                                        # I_1 % 4 != 0: the generic TTM path for the large first contraction
                                        ("c2", (99, 120, 90)),
                                        # wide (J = 60) mode-0 TTM kernel with ragged i and column tails
                                        ("c5", (100, 130, 90))])
def test_rhosvd_parity(krp, name, small):
    cfg = synth.config(name) if small is None else synth.config(name).scaled(small)
    x = synth.tensor(cfg, 0)
    om = synth.omegas(cfg.dims, cfg.R, 0)
    _, _, err_ref, _ = oracle.rhosvd(oracle.as_tensor(x, cfg.dims), om, cfg.ranks)
    Q, core, err = krp.krp_rhosvd(_dev(x), cfg.dims, cfg.ranks, [_dev(o) for o in om], with_error=True)
    _check_factors(Q, cfg.ranks)
    assert core.numel() == int(np.prod(cfg.ranks))
    assert abs(err - err_ref) <= ERR_TOL, (err, err_ref)
    # the returned decomposition reproduces its own error value (oracle reconstruction of GPU factors)
    qs = [q.double().cpu().numpy() for q in Q]
    g = core.double().cpu().numpy().reshape(cfg.ranks, order="F")
    e2 = oracle.tucker_error(oracle.as_tensor(x, cfg.dims), g, qs)
    assert abs(e2 - err) <= 1e-5 + 1e-3 * err


def test_rhosvd_exact_recovery_on_device(krp):
    """Noise-free Tucker tensor with ranks <= targets: relative error at fp32 level."""
    cfg = synth.Config("exact", (96, 80, 64), 12, (6, 6, 6), "tucker", core=(5, 6, 4))
    x = synth.tensor(cfg, 11)
    om = synth.omegas(cfg.dims, cfg.R, 11)
    _, _, err = krp.krp_rhosvd(_dev(x), cfg.dims, cfg.ranks, [_dev(o) for o in om], with_error=True)
    assert err < 1e-5


def _sthosvd_step_checks(krp, x, dims, oms, ranks, Q):
    """Per-step parity (R16): the oracle is fed the GPU's own step input G^(i-1) = X x_1 Q_1^T .. x_{i-1}
    Q_{i-1}^T (built in fp64 from the GPU factors); the GPU's single-mode sketch of that input must match
    the oracle's (1e-5), and the GPU's Q_i must lie in the range of that step sketch."""
    d = len(dims)
    X = oracle.as_tensor(x, dims)
    qs = [q.double().cpu().numpy() for q in Q]
    G = X
    cur = list(dims)
    for i in range(d):
        om_i = [None if j == i else (oms[i][j][:ranks[j]] if j < i else oms[i][j]) for j in range(d)]
        y_ref = oracle.sketch_mode(G, om_i, i)
        gin = np.asarray(G, dtype=np.float64).reshape(-1, order="F").astype(np.float32)
        y_gpu = krp.krp_sketch_mode(_dev(gin), cur, i, [None if o is None else _dev(o) for o in om_i])
        e = rel(y_gpu.cpu().numpy(), oracle.sketch_mode(oracle.as_tensor(gin, cur), om_i, i))
        assert e <= Y_TOL, (i, e)
        # range(Q_i) ⊆ range(Y_i): the residual of projecting Q_i on an orthonormal basis of Y_i
        u, sv, _ = np.linalg.svd(y_ref, full_matrices=False)
        keep = sv > sv[0] * 1e-6
        ub = u[:, keep]
        res = np.linalg.norm(qs[i] - ub @ (ub.T @ qs[i])) / np.sqrt(ranks[i])
        assert res <= 1e-4, (i, res)
        G = oracle.ttm(G, qs[i].T, i)
        cur[i] = ranks[i]


@pytest.mark.parametrize("small", [(32, 32, 32, 32), (40, 36, 32, 30)])
def test_sthosvd_parity(krp, small):
    cfg = synth.config("c3").scaled(small)
    x = synth.tensor(cfg, 0)
    oms = synth.sthosvd_omegas(cfg.dims, cfg.R, 0)
    _, _, err_ref, _ = oracle.sthosvd(oracle.as_tensor(x, cfg.dims), oms, cfg.ranks)
    dom = [[None if o is None else _dev(o) for o in row] for row in oms]
    Q, core, err = krp.krp_sthosvd(_dev(x), cfg.dims, cfg.ranks, dom, with_error=True)
    _check_factors(Q, cfg.ranks)
    assert abs(err - err_ref) <= ERR_TOL, (err, err_ref)
    _sthosvd_step_checks(krp, x, cfg.dims, oms, cfg.ranks, Q)


def test_rhosvd_and_sthosvd_at_the_maximum_order(krp):
    """d = 8, the largest order the boundary accepts (krp.h): rHOSVD (Alg. 7) and STHOSVD (Alg. 8) errors
    match the oracle on a small noisy Tucker tensor with truncation (r < R)."""
    cfg = synth.Config("d8", (6, 5, 4, 4, 3, 3, 3, 4), 3, (2,) * 8, "tucker", core=(2,) * 8, eta=1e-3)
    x = synth.tensor(cfg, 3)
    X = oracle.as_tensor(x, cfg.dims)
    om = synth.omegas(cfg.dims, cfg.R, 3)
    _, _, err_ref, _ = oracle.rhosvd(X, om, cfg.ranks)
    Q, core, err = krp.krp_rhosvd(_dev(x), cfg.dims, cfg.ranks, [_dev(o) for o in om], with_error=True)
    _check_factors(Q, cfg.ranks)
    assert core.numel() == 2 ** 8
    assert abs(err - err_ref) <= ERR_TOL, (err, err_ref)
    g = core.double().cpu().numpy().reshape(cfg.ranks, order="F")
    e2 = oracle.tucker_error(X, g, [q.double().cpu().numpy() for q in Q])
    assert abs(e2 - err) <= 1e-5 + 1e-3 * err
    oms = synth.sthosvd_omegas(cfg.dims, cfg.R, 3)
    _, _, serr_ref, _ = oracle.sthosvd(X, oms, cfg.ranks)
    dom = [[None if o is None else _dev(o) for o in row] for row in oms]
    Qs, _, serr = krp.krp_sthosvd(_dev(x), cfg.dims, cfg.ranks, dom, with_error=True)
    _check_factors(Qs, cfg.ranks)
    assert abs(serr - serr_ref) <= ERR_TOL, (serr, serr_ref)


# ----------------------------------------------------------------- NEXT-1: the paper's Cauchy workload
@pytest.mark.parametrize("r", [4, 8])
def test_cauchy_workload_vs_oracle(krp, r):
    """The Cauchy tensor (a = 2, 1-based) at a reduced n, with no oversampling (R = r):
    the device generator reproduces the host closed form bit for bit; the sketch, RHOSVD-KRP-MEMO and
    RSTHOSVD-KRP match the oracle."""
    cfg = synth.config("cauchy").scaled((40, 36, 32, 30))
    ranks = (r,) * 4
    x = synth.tensor(cfg, 0)
    xd = synth.cauchy_device(cfg.dims)
    assert torch.equal(xd.cpu(), torch.from_numpy(x))
    om = synth.omegas(cfg.dims, r, 0)
    X64 = oracle.as_tensor(x, cfg.dims)
    ref = oracle.sketch_all_modes(X64, om)
    Y = krp.krp_sketch_all_modes(xd, cfg.dims, [_dev(o) for o in om])
    for n in range(4):
        assert rel(Y[n].cpu().numpy(), ref[n]) <= Y_TOL
    _, _, e_ref, _ = oracle.rhosvd(X64, om, ranks)
    Q, core, e = krp.krp_rhosvd(xd, cfg.dims, ranks, [_dev(o) for o in om], with_error=True)
    _check_factors(Q, ranks)
    assert abs(e - e_ref) <= ERR_TOL, (e, e_ref)
    oms = synth.sthosvd_omegas(cfg.dims, r, 0)
    _, _, es_ref, _ = oracle.sthosvd(X64, oms, ranks)
    _, _, es = krp.krp_sthosvd(xd, cfg.dims, ranks, [[None if o is None else _dev(o) for o in row] for row in oms],
                               with_error=True)
    assert abs(es - es_ref) <= ERR_TOL, (es, es_ref)


# ----------------------------------------------------------------- NEXT-2: fresh-Ω KRP and dense-Gaussian baselines
@pytest.mark.parametrize("name,small", [("c2", (64, 48, 40)), ("c4", (16, 12, 10, 9, 8))])
def test_rhosvd_fresh_and_gaussian_vs_oracle(krp, name, small):
    """Alg. 7 read literally (a fresh KRP sequence per mode) and the dense-Gaussian RHOSVD / RSTHOSVD baselines
    (Table 1) against the oracle on the same inputs."""
    cfg = synth.config(name).scaled(small)
    R = min(cfg.R, min(small))
    ranks = tuple(min(r, R) for r in cfg.ranks)
    x = synth.tensor(cfg, 0)
    X64 = oracle.as_tensor(x, cfg.dims)
    steps = synth.rhosvd_fresh_omegas(cfg.dims, R, 0)
    _, _, e_ref, _ = oracle.rhosvd_fresh(X64, steps, ranks)
    Q, core, e = krp.krp_rhosvd_fresh(_dev(x), cfg.dims, ranks, [[None if o is None else _dev(o) for o in row]
                                                              for row in steps], with_error=True)
    _check_factors(Q, ranks)
    assert abs(e - e_ref) <= ERR_TOL, (e, e_ref)
    dense = synth.dense_gaussian(cfg.dims, R, 0)
    _, _, eg_ref, _ = oracle.rhosvd_gaussian(X64, dense, ranks)
    _, _, eg = krp.krp_rhosvd_gaussian(_dev(x), cfg.dims, ranks, [_dev(o) for o in dense], with_error=True)
    assert abs(eg - eg_ref) <= ERR_TOL, (eg, eg_ref)
    dst = synth.dense_gaussian_sthosvd(cfg.dims, ranks, R, 0)
    _, _, es_ref = oracle.sthosvd_gaussian(X64, dst, ranks)
    _, _, es = krp.krp_sthosvd_gaussian(_dev(x), cfg.dims, ranks, [_dev(o) for o in dst], with_error=True)
    assert abs(es - es_ref) <= ERR_TOL, (es, es_ref)


def test_gaussian_sketch_with_kr_matrix_equals_krp_sketch(krp):
    """A dense test matrix equal to the Khatri-Rao product makes the baseline's sketch the KRP sketch: pins the
    explicit unfolding (column order of X_(n)) of the dense path on the device."""
    dims, R = (24, 20, 18, 7), 6
    x = synth.random_tensor(dims, 5, 4)
    om = synth.omegas(dims, R, 5)
    dense = [oracle.kr_for_mode(om, n).astype(np.float32) for n in range(4)]
    ranks = (R,) * 4
    Qg, cg, eg = krp.krp_rhosvd_gaussian(_dev(x), dims, ranks, [_dev(o) for o in dense], with_error=True)
    Qk, ck, ek = krp.krp_rhosvd(_dev(x), dims, ranks, [_dev(o) for o in om], with_error=True)
    assert abs(eg - ek) <= 1e-5 * max(1.0, ek), (eg, ek)
    for a, b in zip(Qg, Qk):  # same sketches -> same Q up to the sketch's rounding
        assert np.abs(np.abs(a.double().cpu().numpy().T @ b.double().cpu().numpy()) - np.eye(R)).max() < 1e-3


# ----------------------------------------------------------------- NEXT-4: Hadamard product of Tucker tensors (Alg. 9)
def test_hadamard_tucker_vs_oracle(krp):
    """Alg. 9 on the device (the product Z = X ∗ Y is never formed) against the oracle's Alg. 9: the same
    approximation error of Z (evaluated in fp64 on the explicit Z), orthonormal factors; and exact recovery
    when every sketch width covers the product's multilinear rank q_n s_n."""
    ns, qs_, ss = (60, 50, 40), (3, 4, 2), (2, 3, 4)
    f, xs, g, ys = synth.hadamard_tucker_inputs(ns, qs_, ss, 5)
    z = oracle.hadamard_tucker_explicit(f, xs, g, ys)
    flat = lambda a: _dev(np.asarray(a).reshape(-1, order="F"))
    for ls, ranks in [((8, 8, 8), (6, 6, 6)), ((6, 12, 8), (6, 12, 8))]:
        om = synth.hadamard_omegas(ns, ls, 6)
        qo, ho = oracle.hadamard_tucker_rhosvd(f, xs, g, ys, ranks, om)
        e_ref = oracle.tucker_error(z, ho, qo)
        Q, core = krp.krp_hadamard_tucker(flat(f), [_dev(a) for a in xs], flat(g), [_dev(u) for u in ys], ranks,
                                          [[None if o is None else _dev(o) for o in row] for row in om])
        _check_factors(Q, ranks)
        qs = [q.double().cpu().numpy() for q in Q]
        h = core.double().cpu().numpy().reshape(ranks, order="F")
        e = oracle.tucker_error(z, h, qs)
        assert abs(e - e_ref) <= ERR_TOL, (ls, e, e_ref)
        if ls == ranks:
            assert e < 1e-5, e


def test_rhosvd_ranks_above_the_multilinear_rank(krp):
    """r_n > rank of the core's unfoldings: the truncation eigenproblem has (numerically) null eigenvalues;
    the factors must still be orthonormal and the exact tensor recovered."""
    dims, R, ranks = (24, 20, 16), 8, (5, 5, 5)
    core = np.random.default_rng(2).standard_normal((2, 2, 2))
    us = [np.linalg.qr(np.random.default_rng(10 + k).standard_normal((n, 2)))[0] for k, n in enumerate(dims)]
    x = oracle.multi_ttm(core, us).reshape(-1, order="F").astype(np.float32)
    om = [_dev(o) for o in synth.omegas(dims, R, 3)]
    Q, g, err = krp.krp_rhosvd(_dev(x), dims, ranks, om, with_error=True)
    _check_factors(Q, ranks)
    assert np.isfinite(g.cpu().numpy()).all()
    assert err <= 1e-6, err
