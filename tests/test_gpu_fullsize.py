"""GPU parity at BASELINE.json's FULL sizes, in the launch configuration bench.py times (caller-provided
workspace, the default plan), against the fp64 oracle on the same seeded inputs.

* Sketch: every element of every Y_n at c2 and c3 (and c4, marked slow) against the oracle's full
  explicit-Khatri-Rao sketch (chunked over the last mode: same terms, fp64); at c5, two rows in every
  128-row block of every mode by the column identity (oracle.sketch_rows_ttv).
* rHOSVD: the reported Tucker error against the oracle's own rHOSVD at c2, c4 and c5 (|Δ| <= 1e-4, reading
  R12), plus a relative bar on the GPU's decomposition (its Q_n and core) evaluated by the fp64 oracle:
  1 % at c2 and c4.  At c5 the target error (~1.1e-6) sits at the relative accuracy of any fp32 sketch of
  the fp32 tensor (~1e-6, the same order as c5's 1e-6 noise), so the directions past the noise floor are
  set by rounding and several answers are correct (R16); the bar there is 20 % (reading R22; measured:
  1.15x the oracle's error, 1.05x with an exact core for the GPU's subspaces).  The GPU's own error value
  must also agree with the fp64 evaluation of its decomposition to 1e-6 (its fp32 evaluation floor).
* STHOSVD (c3): the error against the oracle, and per-step parity with the oracle fed the GPU's own step
  input (R16).
* Factors: Q_nᵀQ_n = I within 1e-6.

Tolerances (BASELINE north_star): per-mode relative Frobenius error of Y_n <= 1e-5."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

Y_TOL = 1e-5
ERR_ABS = 1e-4
ERR_REL = 1e-2
QTQ_TOL = 1e-6


@pytest.fixture(scope="module")
def krp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2507_23207_b200 as krp
    from paper_2507_23207_b200 import build
    build.build()
    yield krp


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def _gpu_sketch(krp, cfg, x, om):
    dev = torch.device("cuda", 0)
    X = torch.from_numpy(x).to(dev)
    O = [torch.from_numpy(o).to(dev) for o in om]
    ws = torch.empty(krp.krp_workspace_bytes(krp.OP_SKETCH_ALL, cfg.dims, cfg.R), dtype=torch.uint8, device=dev)
    Y = [torch.empty((n, cfg.R), dtype=torch.float32, device=dev) for n in cfg.dims]
    krp.krp_sketch_all_modes(X, cfg.dims, O, Y=Y, ws=ws)
    torch.cuda.synchronize()
    out = [y.cpu().numpy() for y in Y]
    del X, O, ws, Y
    torch.cuda.empty_cache()
    return out


def _check_q(Q, ranks):
    for q, r in zip(Q, ranks):
        q = q.double().cpu().numpy()
        dev = np.abs(q.T @ q - np.eye(r)).max()
        assert dev <= QTQ_TOL, dev


def _err_close(err, err_ref):
    assert abs(err - err_ref) <= ERR_ABS, (err, err_ref)
    assert abs(err - err_ref) <= ERR_REL * err_ref, (err, err_ref)


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_sketch_fullsize_elementwise(krp, name):
    cfg = synth.config(name)
    x = synth.tensor(cfg, 0)
    om = synth.omegas(cfg.dims, cfg.R, 0)
    Y = _gpu_sketch(krp, cfg, x, om)
    ref = oracle.sketch_all_modes(oracle.as_tensor(x, cfg.dims), om, chunk=max(1, cfg.dims[-1] // 8))
    for n in range(cfg.d):
        assert np.isfinite(Y[n]).all()
        e = _rel(Y[n], ref[n])
        assert e <= Y_TOL, (name, n, e)


def test_sketch_fullsize_c5_rows_in_every_block(krp):
    cfg = synth.config("c5")
    x = synth.tensor(cfg, 0)
    om = synth.omegas(cfg.dims, cfg.R, 0)
    Y = _gpu_sketch(krp, cfg, x, om)
    rng = np.random.default_rng(7)
    for n in range(cfg.d):
        I = cfg.dims[n]
        rows = []
        for b0 in range(0, I, 128):  # two rows in every 128-row block (first + a random one)
            b1 = min(I, b0 + 128)
            rows += sorted({b0, int(rng.integers(b0, b1))})
        ref = oracle.sketch_rows_ttv(x, cfg.dims, om, n, rows)
        assert np.isfinite(Y[n]).all()
        e = _rel(Y[n][rows], ref)
        assert e <= Y_TOL, (n, e)
        # and every sampled row on its own
        for t, i in enumerate(rows):
            assert _rel(Y[n][i], ref[t]) <= 10 * Y_TOL, (n, i)


@pytest.mark.parametrize("name", ["c2", "c4", "c5"])
def test_rhosvd_fullsize_vs_oracle(krp, name):
    cfg = synth.config(name)
    x = synth.tensor(cfg, 0)
    om = synth.omegas(cfg.dims, cfg.R, 0)
    Q, core, err = krp.krp_rhosvd(torch.from_numpy(x).cuda(), cfg.dims, cfg.ranks,
                                  [torch.from_numpy(o).cuda() for o in om], with_error=True)
    _check_q(Q, cfg.ranks)
    torch.cuda.empty_cache()
    X64 = oracle.as_tensor(x, cfg.dims)
    ch = max(1, cfg.dims[-1] // 16)
    _, _, err_ref, _ = oracle.rhosvd(X64, om, cfg.ranks, chunk=ch)
    assert abs(err - err_ref) <= ERR_ABS, (err, err_ref)
    # the GPU decomposition evaluated in fp64 reaches the oracle's error within the per-config bar (R22)
    qs = [q.double().cpu().numpy() for q in Q]
    g = core.double().cpu().numpy().reshape(cfg.ranks, order="F")
    e64 = oracle.tucker_error(X64, g, qs, chunk=ch)
    rel_bar = 0.2 if name == "c5" else ERR_REL
    assert abs(e64 - err_ref) <= rel_bar * err_ref, (e64, err_ref)
    # and the GPU's fp32-evaluated error lies within that evaluation's floor (R22)
    assert abs(err - e64) <= 1e-6, (err, e64)


def test_sthosvd_fullsize_c3(krp):
    cfg = synth.config("c3")
    x = synth.tensor(cfg, 0)
    oms = synth.sthosvd_omegas(cfg.dims, cfg.R, 0)
    dom = [[None if o is None else torch.from_numpy(o).cuda() for o in row] for row in oms]
    Q, core, err = krp.krp_sthosvd(torch.from_numpy(x).cuda(), cfg.dims, cfg.ranks, dom, with_error=True)
    _check_q(Q, cfg.ranks)
    _, _, err_ref, _ = oracle.sthosvd(oracle.as_tensor(x, cfg.dims), oms, cfg.ranks)
    _err_close(err, err_ref)
    # per-step parity (R16): the oracle sketches the GPU's own step input G^(i-1) = X x_1 Q_1^T .. x_{i-1} Q_{i-1}^T
    d = cfg.d
    qs = [q.double().cpu().numpy() for q in Q]
    G = oracle.as_tensor(x, cfg.dims)
    cur = list(cfg.dims)
    for i in range(d):
        om_i = [None if j == i else (oms[i][j][:cfg.ranks[j]] if j < i else oms[i][j]) for j in range(d)]
        gin = np.asarray(G).reshape(-1, order="F").astype(np.float32)
        y_gpu = krp.krp_sketch_mode(torch.from_numpy(gin).cuda(), cur, i,
                                    [None if o is None else torch.from_numpy(o).cuda() for o in om_i])
        y_ref = oracle.sketch_mode(oracle.as_tensor(gin, cur), om_i, i)
        assert _rel(y_gpu.cpu().numpy(), y_ref) <= Y_TOL, i
        # the GPU's Q_i lies in the range of that step's sketch
        u, sv, _ = np.linalg.svd(y_ref, full_matrices=False)
        ub = u[:, sv > sv[0] * 1e-6]
        assert np.linalg.norm(qs[i] - ub @ (ub.T @ qs[i])) / np.sqrt(cfg.ranks[i]) <= 1e-4, i
        G = oracle.ttm(G, qs[i].T, i)
        cur[i] = cfg.ranks[i]
