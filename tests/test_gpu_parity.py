"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded inputs.

Tolerances (BASELINE north_star): per-mode relative Frobenius error of Y_n <= 1e-5; Tucker relative
error within 1e-4 (absolute difference, reading R12).  Small-integer inputs are exact in 3xTF32 and
fp32, so the worked example is compared bit for bit.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

Y_TOL = 1e-5
ERR_TOL = 1e-4
ENGINES = {"auto": 0, "tc": 1, "simt": 2}


@pytest.fixture(scope="module")
def krp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2507_23207_b200 as krp
    from paper_2507_23207_b200 import build
    build.build()
    yield krp
    krp.krp_set_engine(0)


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _engine_or_skip(krp, engine, fn):
    krp.krp_set_engine(ENGINES[engine])
    try:
        return fn()
    except krp.KrpError as e:
        if e.status == 7 and engine == "tc":
            pytest.skip("shape not tiled by the tcgen05 engine")
        raise
    finally:
        krp.krp_set_engine(0)


# ----------------------------------------------------------------- the sketch
@pytest.mark.parametrize("engine", ["simt", "auto"])
def test_integer_worked_example_bit_exact(krp, engine):
    """Hand-derived example (tests/golden/krp_int_2x2x2.txt): exact on the device."""
    x = np.arange(1, 9, dtype=np.float32)
    om = [np.array([[1, -1], [2, 0]], np.float32), np.array([[0, 1], [1, 2]], np.float32),
          np.array([[1, 1], [-1, 3]], np.float32)]
    ref = oracle.sketch_all_modes(oracle.as_tensor(x, (2, 2, 2)), om)
    krp.krp_set_engine(ENGINES[engine])
    Y = krp.krp_sketch_all_modes(_dev(x), (2, 2, 2), [_dev(o) for o in om])
    krp.krp_set_engine(0)
    for n in range(3):
        assert np.array_equal(Y[n].cpu().numpy(), ref[n].astype(np.float32)), n


SHAPES = [
    ((3, 4, 5), 3), ((2, 3, 4, 5), 4), ((17, 33, 9), 7), ((64, 64, 64), 10), ((130, 7, 64), 5),
    ((256, 129, 3), 16), ((128, 128, 40), 40), ((256, 256, 17), 40), ((384, 128, 9), 64),
    ((16, 16, 16, 16, 16), 20), ((64, 64, 8, 8), 20), ((6, 5, 4, 3, 2, 2), 6), ((1000, 3), 2),
    ((128, 256, 7), 128), ((512, 128, 5), 30),
    # degenerate cases: R = 1, unit modes (first, middle, last), a single-element tensor
    ((128, 128, 128), 1), ((1, 128, 256), 8), ((128, 1, 256), 8), ((256, 128, 1), 8), ((1, 1, 1), 1),
]


@pytest.mark.parametrize("engine", ["simt", "tc", "auto"])
@pytest.mark.parametrize("dims,R", SHAPES)
def test_sketch_all_modes_random(krp, engine, dims, R):
    x = synth.random_tensor(dims, seed=1, tag=len(dims))
    om = synth.omegas(dims, R, seed=2)
    ref = oracle.sketch_all_modes(oracle.as_tensor(x, dims), om)
    Y = _engine_or_skip(krp, engine, lambda: krp.krp_sketch_all_modes(_dev(x), dims, [_dev(o) for o in om]))
    for n in range(len(dims)):
        e = rel(Y[n].cpu().numpy(), ref[n])
        assert e <= Y_TOL, (n, e)


@pytest.mark.parametrize("engine", ["simt", "tc", "auto"])
@pytest.mark.parametrize("dims,R", [((3, 4, 5), 3), ((128, 128, 128), 30), ((20, 128, 128, 8), 30),
                                    ((20, 20, 128, 128), 30), ((20, 20, 20, 128), 30), ((256, 64, 64), 17)])
def test_sketch_single_mode(krp, engine, dims, R):
    x = synth.random_tensor(dims, seed=3, tag=len(dims))
    om = synth.omegas(dims, R, seed=4)
    X = oracle.as_tensor(x, dims)
    for n in range(len(dims)):
        ref = oracle.sketch_mode(X, om, n)
        omn = [None if k == n else _dev(o) for k, o in enumerate(om)]
        Y = _engine_or_skip(krp, engine, lambda: krp.krp_sketch_mode(_dev(x), dims, n, omn))
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


# ----------------------------------------------------------------- rHOSVD / STHOSVD
def _check_factors(Q, ranks):
    for q, r in zip(Q, ranks):
        q = q.double().cpu().numpy()
        assert q.shape[1] == r
        assert np.abs(q.T @ q - np.eye(r)).max() < 1e-4


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


@pytest.mark.parametrize("small", [(32, 32, 32, 32), (40, 36, 32, 30)])
def test_sthosvd_parity(krp, small):
    cfg = synth.config("c3").scaled(small)
    x = synth.tensor(cfg, 0)
    oms = synth.sthosvd_omegas(cfg.dims, cfg.R, 0)
    _, _, err_ref, ys_ref = oracle.sthosvd(oracle.as_tensor(x, cfg.dims), oms, cfg.ranks)
    dom = [[None if o is None else _dev(o) for o in row] for row in oms]
    Q, core, err = krp.krp_sthosvd(_dev(x), cfg.dims, cfg.ranks, dom, with_error=True)
    _check_factors(Q, cfg.ranks)
    assert abs(err - err_ref) <= ERR_TOL, (err, err_ref)
