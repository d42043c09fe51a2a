"""Exact sequential RBM-r' (Algorithm 2)
on the GPU, -m gpu: the dependency-driven sweep (each batch waits for the
earlier batches that share a member) equals the oracle's sequential loop over
the batches (same slot draws, bit-exact; states within the
BASELINE.json tolerances)."""
import numpy as np
import pytest

import rbm_inputs as RI

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1812_10575_b200 import rbm
    rbm.lib()
    return rbm


def E(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


def model(kernel, d, n, p, dtype="f64", **kw):
    kp = {"bounded_confidence": [1.0, 1.0], "coulomb_reg": [0.01]}.get(kernel, [])
    c = dict(d=d, n=n, p=p, dtype=dtype, scheme="rbmr_seq", integrator="em", kernel=kernel, kparam=kp,
             potential="harmonic", vparam=[1.0], constraint="none", sigma=0.1, dt=1e-3, seed=31,
             init="normal", iparam=[0.0, 1.0])
    c.update(kw)
    return c


CASES = [("smooth", 1, 5001, 2), ("smooth", 1, 5001, 3), ("gauss_attr_rep", 2, 20011, 8),
         ("coulomb_reg", 3, 30000, 2), ("coulomb_reg", 3, 1_000_003, 2)]


@pytest.mark.parametrize("kernel,d,n,p", CASES)
def test_seq_slots_and_one_step(R, O, kernel, d, n, p):
    c = model(kernel, d, n, p, step0=2)
    s = R.RBM(c)
    x0 = s.gather(host=True)
    s.step()
    assert np.array_equal(s.slots(), O.rbmr_slots(c, 2))
    assert E(s.gather(host=True), O.rbmr_seq_step(c, x0, 2)) <= 1e-12
    s.close()


def test_seq_split_dyson_and_sphere(R, O):
    c = dict(RI.c1_dyson(n=3000, integrator="split", seed=6), scheme="rbmr_seq")
    s = R.RBM(c)
    x0 = s.gather(host=True)
    s.run(20)
    assert E(s.gather(host=True), O.run(c, x0, 0, 20)) <= 1e-9
    s.close()
    c = dict(RI.c2_sphere(n=20000, seed=2), scheme="rbmr_seq")
    s = R.RBM(c)
    x0 = s.gather(host=True)
    s.step()
    g = s.gather(host=True)
    assert E(g, O.rbmr_seq_step(c, x0, 0)) <= 1e-12
    assert np.max(np.abs(np.linalg.norm(g, axis=1) - 1)) < 1e-14
    s.close()


def test_seq_many_steps_and_fp32(R, O):
    c = model("smooth", 1, 4000, 4)
    s = R.RBM(c)
    x0 = s.gather(host=True)
    s.run(30)
    assert E(s.gather(host=True), O.run(c, x0, 0, 30)) <= 1e-9
    s.close()
    c32 = model("coulomb_reg", 3, 50000, 2, dtype="f32")
    s = R.RBM(c32)
    x0 = s.gather(host=True).astype(np.float64)
    s.step()
    assert E(s.gather(host=True), O.rbmr_seq_step(c32, x0, 0)) <= 1e-4
    s.close()


def test_seq_step_run_and_set_state(R, O):
    """rbm_step x k == rbm_run(k) (graph path) bit-exactly, and a set_state
    between runs (the AoS state and its write counters are rebuilt) continues
    the oracle's trajectory; p = 2 (pair path) and p = 3 (general path)."""
    for p in (2, 3):
        c = model("coulomb_reg", 3, 40_009, p, seed=5)
        a = R.RBM(c)
        b = R.RBM(c)
        x0 = a.gather(host=True)
        for _ in range(6):
            a.step()
        b.run(6)
        ga, gb = a.gather(host=True), b.gather(host=True)
        assert np.array_equal(ga, gb)
        assert E(ga, O.run(c, x0, 0, 6)) <= 1e-10
        b.set_state(gb)
        b.run(4)
        assert E(b.gather(host=True), O.run(c, x0, 0, 10)) <= 1e-9
        a.close()
        b.close()


def test_seq_fp32_pair_path_large(R, O):
    """fp32, p = 2: the sweep's 128-bit record path (position and write
    counter in one access) at N = 2^21 under full occupancy: two runs are
    bit-identical (no ordering race changes a result) and match the oracle's
    sequential loop within the fp32 bound."""
    c = model("coulomb_reg", 3, 1 << 21, 2, dtype="f32", seed=9)
    a = R.RBM(c)
    x0 = a.gather(host=True).astype(np.float64)
    a.run(5)
    g1 = a.gather(host=True)
    a.close()
    b = R.RBM(c)
    b.run(5)
    g2 = b.gather(host=True)
    b.close()
    assert np.array_equal(g1, g2)
    assert E(g1, O.run(c, x0, 0, 5)) <= 1e-4


@pytest.mark.parametrize("scheme", ["rbmr", "rbmr_seq"])
def test_rbmr_widest_partition_layout(R, scheme, monkeypatch):
    """The slot partition at its widest layout (B = 20: 2^10 pass-1 buckets,
    2^10 final buckets each; reached by N >= 2^29 at the default 1024 ids per
    bucket, here by N = 2^27 at 128 ids per bucket) gives results
    bit-identical to the default layout (B = 17): the per-particle order of the
    slots, and so every sum, does not depend on the layout.  (Regression: the
    pass-2 splitter's shared-memory size missed its 128-byte header padding,
    which only the 2^10-segment tile table reached.)"""
    import rbm_inputs as RI
    c = dict(RI.c5_coulomb_reg(n=1 << 27, scheme=scheme), seed=4)
    out = []
    for w in (None, "128"):
        if w:
            monkeypatch.setenv("RBM_RBMR_W", w)
        s = R.RBM(c)
        if w:
            assert s.layout[0] == 20
        s.run(2)
        out.append(s.gather())  # device tensor
        s.sync()
        s.close()
    assert torch.equal(out[0], out[1])


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("scheme", ["rbmr", "rbmr_seq"])
def test_rbmr_two_pass_layout_full_state(R, O, scheme, dtype):
    """C5 physics at N = 4,194,319: the slot partition by particle index takes
    two passes (B = 13 > 10: pass-2 split of the increment / link records, then
    the per-bucket apply / the sweep's chains) -- the layout the C5 RBM-r and
    RBM-r' bench lines time.  Slot draws bit-exact and every particle against
    the oracle (Alg. 2; Jacobi form D:8) at two consecutive
    steps."""
    c = dict(RI.c5_coulomb_reg(n=4_194_319, scheme=scheme), dtype=dtype, seed=9)
    s = R.RBM(c)
    assert s.layout[0] > 10 and s.layout[1] == 2
    step = O.rbmr_step if scheme == "rbmr" else O.rbmr_seq_step
    tol = 1e-12 if dtype == "f64" else 1e-4
    for m in (0, 1):
        x0 = s.gather(host=True).astype(np.float64)
        s.step()
        assert np.array_equal(s.slots(), O.rbmr_slots(c, m))
        assert E(s.gather(host=True), step(c, x0, m)) <= tol
    s.close()


@pytest.mark.parametrize("scheme", ["rbmr", "rbmr_seq"])
def test_rbmr_full_state_large(R, O, scheme):
    """Every particle against the oracle at one eighth of the bench size
    (C5 physics, N = 33,554,399, fp32; slot partition B = 15, two passes):
    slot draws bit-exact, states within the fp32 bar, at two consecutive steps."""
    c = dict(RI.c5_coulomb_reg(n=33_554_399, scheme=scheme), seed=5)
    s = R.RBM(c)
    assert s.layout[0] == 15 and s.layout[1] == 2
    step = O.rbmr_step if scheme == "rbmr" else O.rbmr_seq_step
    for m in (0, 1):
        x0 = s.gather(host=True).astype(np.float64)
        s.step()
        assert np.array_equal(s.slots(), O.rbmr_slots(c, m))
        assert E(s.gather(host=True), step(c, x0, m)) <= 1e-4
    s.close()
