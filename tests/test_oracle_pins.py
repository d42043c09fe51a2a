"""Pins of the CPU oracle against what the paper and mathematics fix.

No CUDA here (-m "not gpu").  Each test names the passage it pins.  The
oracle is never compared with itself: pins are published vectors, closed
forms, exact combinatorial identities (Lemma 3.1), invariants, special cases
and brute force on tiny inputs.
"""
import itertools
import math
import os

import numpy as np
import pytest
from scipy import stats

import rbm_inputs as RI

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def base(**kw):
    c = dict(d=1, n=8, p=2, dtype="f64", scheme="rbm1", integrator="em", kernel="smooth",
             kparam=[], potential="none", vparam=[1.0], constraint="none", sigma=0.0,
             dt=0.01, seed=12345, init="normal", iparam=[0.0, 1.0])
    c.update(kw)
    return c


# ---------------------------------------------------------------- RNG (D:13)
def test_philox_known_answer_vectors(O):
    """Published Philox4x32-10 KAT vectors (tests/golden/philox4x32_10_kat.txt)."""
    rows = [l.split() for l in open(os.path.join(GOLD, "philox4x32_10_kat.txt"))
            if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        v = [int(t, 16) for t in r]
        out = O.philox(v[0:4], v[4:6])
        assert [int(w) for w in out] == v[6:10]


def test_uniform_maps_open_interval_exact(O):
    """D:13: u = (2(w>>9)+1) 2^-24 and (2k+1) 2^-53 lie strictly in (0,1)."""
    assert O.u01_f32(0) == 2.0**-24
    assert O.u01_f32(0xFFFFFFFF) == 1.0 - 2.0**-24
    assert O.u01_f32(0x1FF) == 2.0**-24          # low 9 bits dropped
    assert O.u01_f32(0x200) == 3 * 2.0**-24
    assert O.u01_f64(0, 0) == 2.0**-53
    assert O.u01_f64(0xFFFFFFFF, 0xFFFFFFFF) == 1.0 - 2.0**-53
    assert O.u01_f64(0, 0x1000) == 3 * 2.0**-53


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_noise_is_standard_normal(O, dtype):
    """P:943 z ~ N(0,1): KS test and moments over 60000 draws (d=3)."""
    c = base(d=3, n=4, dtype=dtype)
    z = np.array([O.noise(c, i, m) for i in range(2000) for m in range(10)]).ravel()
    assert abs(z.mean()) < 5 / math.sqrt(z.size)
    assert abs(z.var() - 1) < 5 * math.sqrt(2 / z.size)
    assert stats.kstest(z, "norm").pvalue > 1e-4
    # coordinates are independent
    zz = z.reshape(-1, 3)
    cc = np.corrcoef(zz.T)
    assert np.all(np.abs(cc - np.eye(3)) < 5 / math.sqrt(zz.shape[0]))


def test_noise_depends_on_step_id_replica(O):
    c = base(d=2)
    a = O.noise(c, 3, 7)
    assert not np.array_equal(a, O.noise(c, 4, 7))
    assert not np.array_equal(a, O.noise(c, 3, 8))
    assert not np.array_equal(a, O.noise(dict(c, replica=1), 3, 7))
    assert np.array_equal(a, O.noise(c, 3, 7))


# --------------------------------------------------------------- init
def test_init_normal_moments(O):
    c = base(d=3, n=50000, init="normal", iparam=[0.5, 2.0])
    x = O.init(c)
    assert abs(x.mean() - 0.5) < 5 * 2 / math.sqrt(x.size)
    assert abs(x.std() - 2.0) < 0.02
    assert stats.kstest(((x - 0.5) / 2).ravel(), "norm").pvalue > 1e-4


def test_init_box_uniform(O):
    c = base(d=2, n=50000, init="box", iparam=[-5.0, 5.0])
    x = O.init(c)
    assert x.min() > -5 and x.max() < 5
    assert stats.kstest(x.ravel(), "uniform", args=(-5, 10)).pvalue > 1e-4


def test_init_sphere_uniform(O):
    c = base(d=3, n=50000, init="sphere")
    x = O.init(c)
    assert np.allclose(np.linalg.norm(x, axis=1), 1.0, atol=1e-15)
    # Archimedes: each coordinate of a uniform point on S^2 is U[-1,1]
    assert stats.kstest(x[:, 2], "uniform", args=(-1, 2)).pvalue > 1e-4
    assert np.all(np.abs(x.mean(0)) < 0.02)


def _mixture_parts(O, seed, n, std, K=5, lo=-4.0, hi=4.0):
    """Centres and component labels of the mixture init (D:14): with the
    component std at 1e-12 every point sits on its centre, and neither the
    centres nor the labels depend on the std (their Philox blocks are
    (k, {0,2}, 0, INIT_AUX) and (id, 1, 0, INIT_AUX))."""
    c = base(d=2, n=n, init="mixture", iparam=[K, 1e-12, lo, hi], seed=seed)
    x = O.init(c)
    _, lab = np.unique(np.round(x, 6), axis=0, return_inverse=True)
    lab = lab.ravel()
    cent = np.array([x[lab == k].mean(0) for k in range(lab.max() + 1)])  # within 1e-12 of the centres
    return cent, lab, O.init(dict(c, iparam=[K, std, lo, hi]))


def mixture_pin(O, seeds, n, std_claimed, std_used):
    """Return the p-values of the mixture pins for data drawn with std_used
    while the configuration claims std_claimed (they differ only in the
    deliberately-wrong sensitivity check)."""
    K = 5
    cx, chi2, dof, resid = [], 0.0, 0, []
    for sd in seeds:
        cent, lab, x = _mixture_parts(O, sd, n, std_used, K=K)
        assert cent.shape[0] == K                       # every component drawn
        cx.append(cent)
        cnt = np.bincount(lab, minlength=K)
        chi2 += float(np.sum((cnt - n / K) ** 2 / (n / K)))  # Binomial(n, 1/K) each
        dof += K - 1
        resid.append((x - cent[lab]) / std_claimed)
    cx = np.concatenate(cx)
    r = np.concatenate(resid).ravel()
    return {"centres_x": stats.kstest(cx[:, 0], "uniform", args=(-4.0, 8.0)).pvalue,
            "centres_y": stats.kstest(cx[:, 1], "uniform", args=(-4.0, 8.0)).pvalue,
            "weights": float(stats.chi2.sf(chi2, dof)),
            "resid_normal": stats.kstest(r, "norm").pvalue,
            "resid_std": float(r.std())}


def test_init_mixture_pinned(O):
    """D:14 (BASELINE.json C4: 5 isotropic Gaussians, std 0.5, centres U[-4,4]^2,
    equal weights).  Over 200 seeds: the 1000 centres are U[-4,4] per axis (KS),
    the per-component counts are Binomial(N, 1/5) (chi^2), and the offsets from
    the own centre are N(0, 0.5^2) per coordinate (KS and std)."""
    pv = mixture_pin(O, range(1, 201), 2000, 0.5, 0.5)
    assert pv["centres_x"] > 1e-3 and pv["centres_y"] > 1e-3, pv
    assert pv["weights"] > 1e-3, pv
    assert pv["resid_normal"] > 1e-3 and abs(pv["resid_std"] - 1.0) < 0.01, pv


def test_init_mixture_pin_rejects_wrong_std(O):
    """The pin above fails on a deliberately wrong component std (1.0 drawn,
    0.5 claimed): the residual test must reject it."""
    pv = mixture_pin(O, range(1, 21), 2000, 0.5, 1.0)
    assert pv["resid_normal"] < 1e-6 and abs(pv["resid_std"] - 2.0) < 0.05, pv


def test_init_mixture_offsets_are_the_normal_draws(O):
    """The offset of x_i from its centre is std * z_i with z_i the same
    Brownian-free normal block as the NORMAL init (D:13/D:14):
    mixture(std) - centre == NORMAL(0, std) for every particle."""
    cent, lab, x = _mixture_parts(O, 7, 5000, 0.5)
    z = O.init(base(d=2, n=5000, init="normal", iparam=[0.0, 0.5], seed=7))
    assert np.max(np.abs((x - cent[lab]) - z)) < 1e-11


# ------------------------------------------------------- random division (Alg. 1)
def test_permutation_is_partition(O):
    for n in [1, 2, 7, 100, 1001]:
        c = base(n=n, p=2 if n >= 2 else 1)
        o = O.permutation(c, 5)
        assert np.array_equal(np.sort(o), np.arange(n, dtype=np.uint32))


def test_permutation_sorted_by_key_then_id(O):
    c = base(n=300)
    o = O.permutation(c, 11)
    keys = np.array([O.key(c, int(i), 11) for i in o], dtype=np.uint64)
    comp = keys * (1 << 32) + o.astype(np.uint64)
    assert np.all(comp[1:] > comp[:-1])


def test_division_uniform_n4_p2(O):
    """M(2) = 3 partitions of 4 objects into pairs, each with prob 1/3."""
    c = base(n=4, p=2)
    counts = {}
    T = 30000
    for m in range(T):
        o = O.permutation(c, m)
        part = frozenset([frozenset(o[0:2]), frozenset(o[2:4])])
        counts[part] = counts.get(part, 0) + 1
    assert len(counts) == 3
    for v in counts.values():
        assert abs(v / T - 1 / 3) < 4 * math.sqrt((1 / 3) * (2 / 3) / T)


def test_division_uniform_n6_p3_chi2(O):
    """M(2) = 6!/(3!^2 2!) = 10 partitions of 6 into triples, uniform."""
    c = base(n=6, p=3)
    counts = {}
    T = 30000
    for m in range(T):
        o = O.permutation(c, m)
        part = frozenset([frozenset(o[0:3]), frozenset(o[3:6])])
        counts[part] = counts.get(part, 0) + 1
    assert len(counts) == 10
    obs = np.array(list(counts.values()))
    assert stats.chisquare(obs).pvalue > 1e-4


def test_same_batch_probabilities(O):
    """P:354 P(i,j same batch) = (p-1)/(N-1); P:385-386 triple prob."""
    n, p, T = 8, 4, 20000
    c = base(n=n, p=p)
    pair = 0
    triple = 0
    for m in range(T):
        o = list(O.permutation(c, m))
        pos = {int(v): k // p for k, v in enumerate(o)}
        pair += pos[0] == pos[1]
        triple += pos[0] == pos[1] == pos[2]
    pp = (p - 1) / (n - 1)
    pt = (p - 1) * (p - 2) / ((n - 1) * (n - 2))
    assert abs(pair / T - pp) < 4 * math.sqrt(pp * (1 - pp) / T)
    assert abs(triple / T - pt) < 4 * math.sqrt(pt * (1 - pt) / T)


def test_batch_remainder_rule(O):
    """P:90 'the last batch does not have to have size p'; reading D:7."""
    assert list(O.batch_starts(8, 2)) == [0, 2, 4, 6, 8]
    assert list(O.batch_starts(7, 2)) == [0, 2, 4, 7]        # r=1 joins last full batch
    assert list(O.batch_starts(8, 3)) == [0, 3, 6, 8]        # r=2 forms its own batch
    assert list(O.batch_starts(5, 5)) == [0, 5]
    for n in range(2, 40):
        for p in range(2, n + 1):
            s = np.asarray(O.batch_starts(n, p), dtype=np.int64)
            assert s[0] == 0 and s[-1] == n and np.all(np.diff(s) >= 2)
            assert np.all(np.diff(s) <= p + 1)


# ------------------------------------------------------------ Lemma 3.1
def all_partitions(n, p):
    """All divisions of range(n) into n/p unordered batches of size p, as orders."""
    def rec(rest):
        if not rest:
            yield []
            return
        first = rest[0]
        for comb in itertools.combinations(rest[1:], p - 1):
            batch = (first,) + comb
            rem = [r for r in rest if r not in batch]
            for tail in rec(rem):
                yield list(batch) + tail
    return [np.array(o, dtype=np.uint32) for o in rec(list(range(n)))]


@pytest.mark.parametrize("n,p", [(4, 2), (6, 2), (6, 3), (8, 2), (8, 4)])
def test_lemma31_mean_and_variance_by_enumeration(O, n, p):
    """E chi = 0 and Var chi = (1/(p-1) - 1/(N-1)) Lambda_i, over ALL M(n) divisions."""
    parts = all_partitions(n, p)
    M = math.factorial(n) // (math.factorial(p) ** (n // p) * math.factorial(n // p))
    assert len(parts) == M
    rng = np.random.default_rng(n * 10 + p)
    for kern, d in [("smooth", 1), ("coulomb_reg", 3), ("gauss_attr_rep", 2)]:
        c = base(n=n, p=p, d=d, kernel=kern, kparam=[0.01])
        x = rng.standard_normal((n, d))
        fs = np.array([O.batch_forces(c, x, o) for o in parts])
        # full mean-field force 1/(N-1) sum_{j != i} K(x_i - x_j): the p=N batch
        cN = dict(c, p=n)
        full = O.batch_forces(cN, x, np.arange(n, dtype=np.uint32))
        assert np.max(np.abs(fs.mean(0) - full)) < 1e-13
        # Lambda_i from K values
        Kij = np.zeros((n, n, d))
        for i in range(n):
            for j in range(n):
                if i != j:
                    Kij[i, j] = O.kernel_eval(c, x[i] - x[j])
        lam = np.zeros(n)
        for i in range(n):
            dev = [Kij[i, j] - full[i] for j in range(n) if j != i]
            lam[i] = sum(float(v @ v) for v in dev) / (n - 2)
        var = ((fs - full) ** 2).sum(-1).mean(0)
        pred = (1 / (p - 1) - 1 / (n - 1)) * lam
        assert np.allclose(var, pred, rtol=1e-11, atol=1e-14)


# ------------------------------------------------------------- forces and models
def test_dyson_virial_identity(O):
    """K=1/x: sum_i x_i F_i = sum_B |B|/2 = N/2 for ANY division (derived from P:889-892)."""
    rng = np.random.default_rng(3)
    for n, p in [(10, 2), (11, 4), (64, 8), (9, 9)]:
        c = base(n=n, p=p, kernel="dyson")
        x = rng.standard_normal((n, 1))
        o = rng.permutation(n).astype(np.uint32)
        f = O.batch_forces(c, x, o)
        assert abs(float((x * f).sum()) - n / 2) < 1e-11


def test_coulomb_virial_identity(O):
    """K=x/|x|^3: sum_i x_i.F_i = sum_B 1/(|B|-1) sum_{pairs in B} 1/r_ij."""
    rng = np.random.default_rng(4)
    n, p = 12, 3
    c = base(n=n, p=p, d=3, kernel="coulomb")
    x = rng.standard_normal((n, 3))
    o = rng.permutation(n).astype(np.uint32)
    f = O.batch_forces(c, x, o)
    want = 0.0
    for b in range(n // p):
        mem = o[b * p:(b + 1) * p]
        for a, bb in itertools.combinations(mem, 2):
            want += 1.0 / np.linalg.norm(x[a] - x[bb]) / (p - 1)
    assert abs(float((x * f).sum()) - want) < 1e-12


def test_kernel_shapes_closed_forms(O):
    # K4 (BASELINE C4) changes sign where e^{-r^2/2} = e^{-r^2/8}/4: r^2 = 8 ln 4 / 3
    c4 = base(d=2, kernel="gauss_attr_rep")
    r0 = math.sqrt(8 * math.log(4) / 3)
    assert O.kernel_eval(c4, [r0 * (1 - 1e-6), 0])[0] > 0   # repulsive inside
    assert O.kernel_eval(c4, [r0 * (1 + 1e-6), 0])[0] < 0   # attractive beyond
    assert abs(O.kernel_eval(c4, [0, r0])[1]) < 1e-15
    # K5 (BASELINE C5) is bounded, max |K| = sqrt(e/2)/(3e/2)^{3/2} at r = sqrt(e/2)
    eps = 0.01
    c5 = base(d=3, kernel="coulomb_reg", kparam=[eps])
    rs = np.linspace(1e-4, 1.0, 20001)
    mags = [np.linalg.norm(O.kernel_eval(c5, [r, 0, 0])) for r in rs[::50]]
    kmax = math.sqrt(eps / 2) / (1.5 * eps) ** 1.5
    assert abs(np.linalg.norm(O.kernel_eval(c5, [0, 0, math.sqrt(eps / 2)])) - kmax) < 1e-12
    assert max(mags) <= kmax * (1 + 1e-12)
    assert abs(kmax - 38.49) < 0.01
    # K6: max |K| = 1/2 at |z| = 1
    c6 = base(kernel="smooth")
    assert abs(O.kernel_eval(c6, [1.0])[0] - 0.5) < 1e-16
    # K3 (Eq. 5.12, D:10): strict window |z| < r, attraction -alpha z inside
    c3 = base(kernel="bounded_confidence", kparam=[2.0, 1.0])
    assert O.kernel_eval(c3, [1.0])[0] == 0.0
    assert O.kernel_eval(c3, [-1.0])[0] == 0.0
    assert O.kernel_eval(c3, [np.nextafter(1.0, 0)])[0] < 0
    assert O.kernel_eval(c3, [0.5])[0] == -1.0
    # oddness of every registry kernel
    rng = np.random.default_rng(0)
    for k, d, kp in [("dyson", 1, []), ("coulomb", 3, []), ("bounded_confidence", 1, [1, 1]),
                     ("gauss_attr_rep", 2, []), ("coulomb_reg", 3, [0.01]), ("smooth", 1, [])]:
        c = base(d=d, kernel=k, kparam=kp)
        for _ in range(20):
            z = rng.standard_normal(d)
            assert np.array_equal(O.kernel_eval(c, z), -O.kernel_eval(c, -z))
    # singular kernels at coincident points (D:12)
    assert O.kernel_eval(base(kernel="dyson"), [0.0])[0] == 0.0
    assert np.all(O.kernel_eval(base(d=3, kernel="coulomb"), [0, 0, 0]) == 0.0)


def test_bounded_confidence_fp32_window(O):
    """D:10: in fp32 mode the window is tested on fl32(x_i - x_j)."""
    a = np.float32(0.7)
    b = np.float32(-0.3000000119)       # exact difference just above 1 in fp64? check fp32
    c32 = base(n=2, p=2, kernel="bounded_confidence", kparam=[1.0, 1.0], dtype="f32")
    c64 = dict(c32, dtype="f64")
    x = np.array([[float(a)], [float(b)]])
    d32 = np.float32(a) - np.float32(b)
    d64 = float(a) - float(b)
    f32 = O.batch_forces(c32, x, np.array([0, 1], dtype=np.uint32))
    f64 = O.batch_forces(c64, x, np.array([0, 1], dtype=np.uint32))
    assert (f32[0, 0] != 0) == (abs(float(d32)) < 1.0)
    assert (f64[0, 0] != 0) == (abs(d64) < 1.0)


# ---------------------------------------------------------------- one step
def test_em_closed_form_harmonic(O):
    """K=0, V=|x|^2/2, sigma=0: x' = x - dt x (P:819 forward Euler)."""
    c = base(n=50, p=5, d=3, kernel="zero", potential="harmonic", dt=0.01)
    x = np.random.default_rng(1).standard_normal((50, 3))
    y = O.rbm1_step(c, x, 0)
    assert np.allclose(y, (1 - 0.01) * x, rtol=0, atol=1e-15)


def test_em_two_particles_smooth(O):
    """N=2, K6, (0,1), dt=0.1, Euler: (-0.05, 1.05) under Eq. 1.2's sign."""
    c = base(n=2, p=2, kernel="smooth", dt=0.1)
    y = O.rbm1_step(c, np.array([[0.0], [1.0]]), 0)
    assert np.allclose(y.ravel(), [-0.05, 1.05], atol=1e-15)


def test_p_equals_n_is_direct_step(O):
    """p=N: the single batch is the full system (chi == 0)."""
    rng = np.random.default_rng(2)
    for kern, d, kp, pot, sig in [("smooth", 1, [], "harmonic", 0.3), ("coulomb_reg", 3, [0.01], "harmonic", 0.1),
                                  ("gauss_attr_rep", 2, [], "none", 0.05)]:
        n = 37
        c = base(n=n, p=n, d=d, kernel=kern, kparam=kp, potential=pot, sigma=sig)
        x = rng.standard_normal((n, d))
        a = O.rbm1_step(c, x, 4)
        b = O.direct_step(c, x, 4)
        assert np.max(np.abs(a - b)) < 1e-14


def test_momentum_conserved(O):
    """V=0, sigma=0, odd K: every batch conserves sum_i x_i (Eq. 2.2)."""
    rng = np.random.default_rng(5)
    for kern, d, kp in [("bounded_confidence", 1, [1.0, 1.0]), ("gauss_attr_rep", 2, []),
                        ("coulomb_reg", 3, [0.01]), ("smooth", 1, []), ("coulomb", 3, [])]:
        for n, p in [(64, 2), (63, 4), (40, 8)]:
            c = base(n=n, p=p, d=d, kernel=kern, kparam=kp)
            x = rng.standard_normal((n, d))
            y = O.rbm1_step(c, x, 9)
            assert np.max(np.abs(y.sum(0) - x.sum(0))) < 1e-12


def test_noise_mean_shift_exact(O):
    """C3 with sigma>0: mean(x') - mean(x) = sigma sqrt(dt) mean(z) (momentum + noise)."""
    cfg = RI.c3_opinion(n=1000)
    cfg["dtype"] = "f64"
    x = O.init(cfg)
    y = O.rbm1_step(cfg, x, 3)
    z = np.array([O.noise(cfg, i, 3) for i in range(1000)])
    assert abs((y - x).mean() - cfg["sigma"] * math.sqrt(cfg["dt"]) * z.mean()) < 1e-15


def test_opinion_range_monotone(O):
    """D:10 model with sigma=0: each pair moves toward its midpoint, so min/max are monotone."""
    cfg = dict(RI.c3_opinion(n=2000), sigma=0.0, dtype="f64")
    x = O.init(cfg)
    lo, hi = x.min(), x.max()
    for m in range(50):
        x = O.rbm1_step(cfg, x, m)
        assert x.min() >= lo - 1e-15 and x.max() <= hi + 1e-15
        lo, hi = x.min(), x.max()


# -------------------------------------------------------- split pair flows (D:3)
def rk4_pair(O, c, xi, xj, tau, nsub=2000):
    h = tau / nsub
    def f(a, b):
        return O.kernel_eval(c, a - b), O.kernel_eval(c, b - a)
    a, b = np.array(xi, float), np.array(xj, float)
    for _ in range(nsub):
        k1a, k1b = f(a, b)
        k2a, k2b = f(a + h / 2 * k1a, b + h / 2 * k1b)
        k3a, k3b = f(a + h / 2 * k2a, b + h / 2 * k2b)
        k4a, k4b = f(a + h * k3a, b + h * k3b)
        a = a + h / 6 * (k1a + 2 * k2a + 2 * k3a + k4a)
        b = b + h / 6 * (k1b + 2 * k2b + 2 * k3b + k4b)
    return a, b


@pytest.mark.parametrize("tau", [1e-3, 1e-2])
def test_dyson_pair_flow_vs_rk4(O, tau):
    """P:922-943 exact flow (with the 1/2 of D:3) solves dX^i = K(X^i-X^j)dt."""
    c = base(kernel="dyson")
    rng = np.random.default_rng(6)
    for _ in range(5):
        xi, xj = rng.standard_normal(1), rng.standard_normal(1)
        yi, yj = O.pair_flow(c, xi, xj, tau)
        ri, rj = rk4_pair(O, c, xi, xj, tau)
        assert np.max(np.abs(yi - ri)) < 1e-9 and np.max(np.abs(yj - rj)) < 1e-9
        assert abs((yi - yj)[0] ** 2 - (xi - xj)[0] ** 2 - 4 * tau) < 1e-12
        assert abs((yi + yj)[0] - (xi + xj)[0]) < 1e-15
        assert np.sign(yi - yj) == np.sign(xi - xj)
    # the paper's displayed formula without 1/2 would move (0,1) to -0.5198 at tau=0.01
    yi, yj = O.pair_flow(c, [0.0], [1.0], 0.01)
    assert abs(yi[0] - (-0.009901951)) < 1e-9


@pytest.mark.parametrize("tau", [1e-3, 1e-2])
def test_coulomb_pair_flow_vs_rk4(O, tau):
    """P:1029-1045 exact flow: |D|^3 -> |D|^3 + 6 tau, midpoint preserved (D:3)."""
    c = base(d=3, kernel="coulomb")
    rng = np.random.default_rng(7)
    for _ in range(4):
        xi, xj = rng.standard_normal(3), rng.standard_normal(3)
        yi, yj = O.pair_flow(c, xi, xj, tau)
        ri, rj = rk4_pair(O, c, xi, xj, tau)
        assert np.max(np.abs(yi - ri)) < 1e-9 and np.max(np.abs(yj - rj)) < 1e-9
        assert abs(np.linalg.norm(yi - yj) ** 3 - np.linalg.norm(xi - xj) ** 3 - 6 * tau) < 1e-12
        assert np.max(np.abs(yi + yj - xi - xj)) < 1e-15


# ------------------------------------------------------- long-run physics pins
def semicircle_cdf(x):
    x = np.clip(x, -math.sqrt(2), math.sqrt(2))
    return 0.5 + x * np.sqrt(np.maximum(2 - x * x, 0.0)) / (2 * math.pi) + np.arcsin(np.clip(x / math.sqrt(2), -1, 1)) / math.pi


def w1_to_cdf(sample, cdf, lo=-3.0, hi=3.0, m=60001):
    g = np.linspace(lo, hi, m)
    s = np.sort(sample)
    emp = np.searchsorted(s, g, side="right") / s.size
    return float(np.trapezoid(np.abs(emp - cdf(g)), g))


def test_dyson_split_reaches_semicircle(O):
    """P:904-906 equilibrium rho = sqrt(2-x^2)/pi; split RBM-1, N=500, T=10 (D:16, D:17)."""
    w = []
    for seed in [1, 2]:
        cfg = RI.c1_dyson(n=500, integrator="split", seed=seed)
        x = O.init(cfg)
        x = O.run(cfg, x, 0, 10000)
        w.append(w1_to_cdf(x.ravel(), semicircle_cdf))
    assert max(w) < 0.02, w


def test_dyson_second_moment_identity(O):
    """m2(t) = (1+s^2)/2 + (m2(0)-(1+s^2)/2) e^{-2t} (derived from Eq. 1.2 with K=1/x)."""
    cfg = RI.c1_dyson(n=4000, integrator="split", seed=3)
    x = O.init(cfg)
    s2 = cfg["sigma"] ** 2
    m20 = float((x ** 2).mean())
    x = O.run(cfg, x, 0, 1000)
    pred = (1 + s2) / 2 + (m20 - (1 + s2) / 2) * math.exp(-2.0)
    assert abs(float((x ** 2).mean()) - pred) < 0.01


def thomson_energy(x):
    e = 0.0
    for i in range(len(x)):
        for j in range(i + 1, len(x)):
            e += 1.0 / np.linalg.norm(x[i] - x[j])
    return e


def thomson_minimum(n):
    """Closed-form minimal configurations (antipodes, triangle, tetrahedron,
    triangular bipyramid, octahedron, icosahedron)."""
    s3 = math.sqrt(3)
    if n == 2:
        pts = [[0, 0, 1], [0, 0, -1]]
    elif n == 3:
        pts = [[1, 0, 0], [-0.5, s3 / 2, 0], [-0.5, -s3 / 2, 0]]
    elif n == 4:
        pts = [[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]]
    elif n == 5:
        pts = [[0, 0, 1], [0, 0, -1], [1, 0, 0], [-0.5, s3 / 2, 0], [-0.5, -s3 / 2, 0]]
    elif n == 6:
        pts = [[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]]
    elif n == 12:
        ph = (1 + math.sqrt(5)) / 2
        pts = []
        for a in (-1, 1):
            for b in (-ph, ph):
                pts += [[0, a, b], [a, b, 0], [b, 0, a]]
    pts = np.array(pts, float)
    pts /= np.linalg.norm(pts, axis=1, keepdims=True)
    return thomson_energy(pts)


def test_thomson_closed_forms_sanity():
    assert abs(thomson_minimum(2) - 0.5) < 1e-14
    assert abs(thomson_minimum(3) - math.sqrt(3)) < 1e-14
    assert abs(thomson_minimum(4) - 3.674234614) < 1e-8
    assert abs(thomson_minimum(6) - 9.985281374) < 1e-8
    assert abs(thomson_minimum(12) - 49.165253058) < 1e-8


@pytest.mark.parametrize("n", [4, 6, 12])
def test_thomson_small_n_reaches_minimum(O, n):
    """Sec. 5.1: RBM with p=2 on the sphere finds the ground
    state; annealed dt then a p=N polish lands on the closed-form minimum."""
    cfg = RI.c2_sphere(n=n, seed=n)
    x = O.init(cfg)
    m = 0
    for dt, T in [(1e-2, 60.0), (3e-3, 60.0), (1e-3, 60.0)]:
        c = dict(cfg, dt=dt)
        k = int(round(T / dt))
        x = O.run(c, x, m, k)
        m += k
    assert np.allclose(np.linalg.norm(x, axis=1), 1.0, atol=1e-12)
    e_rbm = thomson_energy(x)
    emin = thomson_minimum(n)
    assert (e_rbm - emin) / emin < 2e-3
    c = dict(cfg, p=n, dt=5e-2)
    x = O.run(c, x, m, 20000)
    assert abs(thomson_energy(x) - emin) / emin < 1e-8


# ---------------------------------------------------------------- RBM-r (D:8, D:9)
def test_rbmr_slots_distinct_and_uniform(O):
    cfg = base(n=4, p=2, scheme="rbmr")
    cnt = {}
    T = 6000
    for m in range(T):
        js = O.rbmr_slots(cfg, m)
        for b in range(2):
            pr = tuple(sorted(js[2 * b:2 * b + 2]))
            assert pr[0] != pr[1]
            cnt[pr] = cnt.get(pr, 0) + 1
    assert len(cnt) == 6
    tot = sum(cnt.values())
    for v in cnt.values():
        assert abs(v / tot - 1 / 6) < 4 * math.sqrt((1 / 6) * (5 / 6) / tot)


def test_rbmr_membership_binomial(O):
    n, p = 1000, 4
    cfg = base(n=n, p=p, scheme="rbmr")
    js = np.concatenate([O.rbmr_slots(cfg, m) for m in range(20)])
    c = np.bincount(js, minlength=n)
    assert abs(c.mean() - 20 * 1.0) < 1e-9        # n*p = N slots per sweep, mean 1
    assert abs(c.var() / 20 - 1.0) < 0.15          # ~Binomial(N, 1/N) per sweep


def test_rbmr_jacobi_matches_rbm1_dynamics(O):
    """RBM-r with N/p iterations per tau tracks RBM-1 (m2 of Dyson split)."""
    m2 = {}
    for scheme in ["rbm1", "rbmr"]:
        cfg = RI.c1_dyson(n=2000, integrator="split", scheme=scheme, seed=5)
        x = O.init(cfg)
        x = O.run(cfg, x, 0, 1000)
        m2[scheme] = float((x ** 2).mean())
    assert abs(m2["rbm1"] - m2["rbmr"]) < 0.02


def test_rbmr_conserves_momentum_when_kernel_only(O):
    """Each slot increment pair of an odd K sums to zero (Jacobi reading D:8)."""
    cfg = base(n=100, p=4, d=2, scheme="rbmr", kernel="gauss_attr_rep")
    x = np.random.default_rng(8).standard_normal((100, 2))
    y = O.rbmr_step(cfg, x, 2)
    assert np.max(np.abs(y.sum(0) - x.sum(0))) < 1e-12


def test_sphere_stays_on_sphere(O):
    cfg = RI.c2_sphere(n=300)
    x = O.init(cfg)
    x = O.run(cfg, x, 0, 20)
    assert np.allclose(np.linalg.norm(x, axis=1), 1.0, atol=1e-14)


# ----------------------------------------------------- wealth model (row f4)
def inv_gamma2_cdf(y, beta):
    """Inverse-Gamma(shape 2, scale beta) CDF: e^{-beta/y} (1 + beta/y) (P:1155-1158
    with kappa = D = 1: rho = beta^2 y^{-3} e^{-beta/y})."""
    y = np.maximum(np.asarray(y, np.float64), 1e-300)
    return np.exp(-beta / y) * (1.0 + beta / y)


def test_linear_pair_flow_closed_form_and_rk4(O):
    """Wealth trading pair flow: D' = D e^{-2 kappa tau}, midpoint kept."""
    c = RI.wealth(n=2, kappa=0.7)
    xi, xj = np.array([2.5]), np.array([-0.5])
    for tau in (1e-3, 0.1, 1.0):
        yi, yj = O.pair_flow(c, xi, xj, tau)
        assert abs((yi - yj)[0] - 3.0 * math.exp(-1.4 * tau)) < 1e-14
        assert abs((yi + yj)[0] - 2.0) < 1e-14
    # RK4 of dxi = -k(xi-xj), dxj = -k(xj-xi)
    a, b, k, h = 2.5, -0.5, 0.7, 1e-3
    for _ in range(1000):
        def f(u, v):
            return -k * (u - v), -k * (v - u)
        k1 = f(a, b); k2 = f(a + h / 2 * k1[0], b + h / 2 * k1[1])
        k3 = f(a + h / 2 * k2[0], b + h / 2 * k2[1]); k4 = f(a + h * k3[0], b + h * k3[1])
        a += h / 6 * (k1[0] + 2 * k2[0] + 2 * k3[0] + k4[0])
        b += h / 6 * (k1[1] + 2 * k2[1] + 2 * k3[1] + k4[1])
    yi, yj = O.pair_flow(c, xi, xj, 1.0)
    assert abs(yi[0] - a) < 1e-10 and abs(yj[0] - b) < 1e-10


def test_geometric_noise_step_is_exact_gbm(O):
    """Split second half with multiplicative noise: x' = y exp(s sqrt(t) z - s^2 t/2),
    the exact GBM step: mean factor 1, log-factor variance s^2 t (checked on
    one split step of a pair with equal members, so the pair flow is the identity)."""
    c = dict(RI.wealth(n=2), dt=0.04)
    s2t = c["sigma"] ** 2 * c["dt"]
    logs = []
    for m in range(4000):
        x = np.array([[1.0], [1.0]])
        y = O.rbm1_step(c, x, m)
        logs.extend(np.log(y.ravel()))
        z = np.array([O.noise(c, i, m)[0] for i in range(2)])
        assert np.allclose(y.ravel(), np.exp(math.sqrt(s2t) * z - 0.5 * s2t), rtol=1e-14)
    logs = np.array(logs)
    assert abs(logs.mean() + 0.5 * s2t) < 4 * math.sqrt(s2t / logs.size)
    assert abs(logs.var() / s2t - 1.0) < 0.06
    assert abs(np.exp(logs).mean() - 1.0) < 4 * math.sqrt((math.exp(s2t) - 1) / logs.size)


def test_linear_em_conserves_pair_sums(O):
    c = dict(RI.wealth(n=1000, integrator="em"), sigma=0.0)
    x = O.init(c)
    y = O.rbm1_step(c, x, 0)
    assert abs(x.sum() - y.sum()) < 1e-10
    # EM with multiplicative noise: x' = x - k dt (x - x_theta) + s x sqrt(dt) z
    c2 = RI.wealth(n=2, integrator="em")
    x = np.array([[1.5], [0.25]])
    y = O.rbm1_step(c2, x, 3)
    z = [O.noise(c2, i, 3)[0] for i in range(2)]
    sq = c2["sigma"] * math.sqrt(c2["dt"])
    assert abs(y[0, 0] - (1.5 - 1e-3 * 1.25 + sq * 1.5 * z[0])) < 1e-15
    assert abs(y[1, 0] - (0.25 + 1e-3 * 1.25 + sq * 0.25 * z[1])) < 1e-15


def test_wealth_reaches_inverse_gamma(O):
    """Fig. wealth: RBM-1, p=2, splitting, tau=1e-3, T=3 from
    X_0 = |N(0,1)|: the empirical law matches the inverse-Gamma equilibrium
    (shape kappa/D+1 = 2, scale kappa eta/D) with eta = sqrt(2/pi) the mean wealth."""
    c = RI.wealth(n=20_000, seed=2)
    x = O.init(c)
    eta = math.sqrt(2.0 / math.pi)
    assert abs(x.mean() - eta) < 4 * math.sqrt((1 - 2 / math.pi) / c["n"])
    x = O.run(c, x, 0, 3000).ravel()
    s = np.sort(x)
    ks = np.max(np.abs(np.arange(1, s.size + 1) / s.size - inv_gamma2_cdf(s, eta)))
    assert ks < 0.03, ks
    assert np.all(x > 0)


# ------------------------------------- exact sequential RBM-r' (row f2, Alg. 2)
def test_rbmr_seq_single_batch_equals_jacobi(O):
    """p = N: one batch per sweep, so Algorithm 2's sequential update and the
    Jacobi sweep (D:8) are the same map (two independent code paths)."""
    c = dict(RI.smooth_test(40, p=40), sigma=0.3, scheme="rbmr_seq")
    x = O.init(c)
    a = O.rbmr_seq_step(c, x, 5)
    b = O.rbmr_step(dict(c, scheme="rbmr"), x, 5)
    assert np.max(np.abs(a - b)) < 1e-14


def test_rbmr_seq_conserves_momentum_and_differs_from_jacobi(O):
    c = dict(RI.smooth_test(1000, p=4), potential="none", sigma=0.0, scheme="rbmr_seq")
    x = O.init(c)
    y = O.rbmr_seq_step(c, x, 0)
    assert abs(y.sum() - x.sum()) < 1e-11  # each batch conserves its sum (odd K, V = 0)
    j = O.rbmr_step(dict(c, scheme="rbmr"), x, 0)
    assert np.max(np.abs(y - j)) > 1e-6     # later batches see earlier updates


def test_rbmr_seq_dyson_second_moment(O):
    """P:200 (N/p iterations ~ time tau): the sequential sweep reproduces the
    Dyson m2(t) closed form like RBM-1 (split, N = 2000, T = 1)."""
    c = dict(RI.c1_dyson(n=2000, integrator="split", seed=4), scheme="rbmr_seq")
    x = O.init(c)
    s2 = c["sigma"] ** 2
    m20 = float((x ** 2).mean())
    x = O.run(c, x, 0, 1000)
    pred = (1 + s2) / 2 + (m20 - (1 + s2) / 2) * math.exp(-2.0)
    assert abs(float((x ** 2).mean()) - pred) < 0.02


# -------------------------------------- second-order RBM, Verlet (row f3)
def verlet_cfg(n, p=2, kernel="smooth", beta=0.0, dt=2.0 ** -7, seed=1):
    """The paper's 1-D Hamiltonian test: X' = V, V' = mean K, stored
    as d = 2 components (x, v) at the start, (x_n, x_{n-1}) after."""
    return dict(d=2, n=n, p=p, dtype="f64", scheme="rbm1", integrator="verlet", kernel=kernel,
                kparam=[], potential="harmonic" if beta else "none", vparam=[beta], constraint="none",
                sigma=0.0, dt=dt, seed=seed, init="user", iparam=[], state_form="xv")


def test_verlet_harmonic_closed_form(O):
    """K = 0, V = beta x^2/2: the Verlet recurrence has the closed-form solution
    x_n = A cos(n th) + B sin(n th), cos th = 1 - beta tau^2 / 2, with x_0 and
    x_1 = x_0 + v_0 tau - beta x_0 tau^2 / 2."""
    beta, tau, n = 2.0, 0.01, 1000
    c = dict(verlet_cfg(3, kernel="zero", beta=beta, dt=tau), p=3)
    x0 = np.array([[1.0, 0.0], [-0.5, 2.0], [0.25, -1.0]])
    y = O.direct_run(c, x0, 0, n)
    th = math.acos(1 - beta * tau * tau / 2)
    for i in range(3):
        a = x0[i, 0]
        x1 = x0[i, 0] + x0[i, 1] * tau - 0.5 * beta * x0[i, 0] * tau * tau
        b = (x1 - a * math.cos(th)) / math.sin(th)
        want = [a * math.cos(n * th) + b * math.sin(n * th), a * math.cos((n - 1) * th) + b * math.sin((n - 1) * th)]
        assert np.allclose(y[i], want, atol=1e-11)
    z = O.run(c, x0, 0, n)  # RBM with p = N: the same map
    assert np.max(np.abs(z - y)) < 1e-12


def test_verlet_p_equals_n_and_momentum(O):
    rng = np.random.default_rng(3)
    n = 60
    x0 = np.stack([RI.semicircle_x0(n, seed=3).ravel(), rng.standard_normal(n)], axis=1)
    c = verlet_cfg(n, p=n)
    a = O.run(c, x0, 0, 50)
    b = O.direct_run(c, x0, 0, 50)
    assert np.max(np.abs(a - b)) < 1e-12
    c2 = verlet_cfg(n, p=2)
    y = O.run(c2, x0, 0, 50)
    # V = 0, odd K: total momentum sum_i (x_n - x_{n-1}) / tau stays sum_i v_0 + O(tau) start term
    p50 = (y[:, 0] - y[:, 1]).sum()
    y51 = O.run(dict(c2, state_form="xx"), y, 50, 1)
    assert abs((y51[:, 0] - y51[:, 1]).sum() - p50) < 1e-12


def test_verlet_rbm_error_decreases_with_tau(O):
    """Fig. second on a small system: RBM-1 (p = 2) Verlet against the
    full-force Verlet reference (tau = 2^-13) at T = 1; the error shrinks with tau."""
    n = 100
    rng = np.random.default_rng(7)
    x0 = np.stack([RI.semicircle_x0(n, seed=7).ravel(), rng.standard_normal(n)], axis=1)
    ref = O.direct_run(verlet_cfg(n, dt=2.0 ** -13), x0, 0, 2 ** 13)
    errs = []
    for k in (4, 7):
        y = O.run(verlet_cfg(n, dt=2.0 ** -k, seed=11), x0, 0, 2 ** k)
        errs.append(float(np.sqrt(np.mean((y[:, 0] - ref[:, 0]) ** 2))))
    assert errs[1] < 0.6 * errs[0], errs


def test_bounded_confidence_closed_window(O):
    """phi = chi_[0,1] is closed -- partners exactly r apart interact;
    the strict window (BASELINE C3, D:10) excludes them."""
    for dtype in ("f64", "f32"):
        base = dict(RI.opinion_paper(n=2, dtype=dtype), dt=0.01)
        z = np.array([1.0])
        closed = O.kernel_eval(base, z)
        strict = O.kernel_eval(dict(base, kparam=[40.0, 1.0, 0.0]), z)
        assert closed[0] == -40.0 and strict[0] == 0.0
        x = np.array([[0.0], [1.0]])
        y = O.rbm1_step(base, x, 0)
        assert np.allclose(y.ravel(), [0.4, 0.6], atol=1e-15)  # x -+ dt * 40 * 1


# ------------------------- clustering through the particle system (Sec. 5.3)
def _tiny_graph():
    """n = 5, symmetric weighted adjacency (a_ij >= 0) in CSR and dense."""
    dense = np.zeros((5, 5))
    for i, j, a in [(0, 1, 1.0), (0, 2, 0.3), (1, 3, 2.0), (2, 4, 0.5), (3, 4, 1.0), (0, 4, 0.1)]:
        dense[i, j] = dense[j, i] = a
    rows, cols = np.nonzero(dense)
    rp = np.zeros(6, dtype=np.uint32)
    np.cumsum(np.bincount(rows, minlength=5), out=rp[1:])
    return (rp, cols.astype(np.uint32), dense[rows, cols]), dense


def _adj_cfg(**kw):
    adj, _ = _tiny_graph()
    c = dict(d=2, n=5, p=2, dtype="f64", scheme="rbmr", integrator="split", kernel="adjacency",
             kparam=[40.0, 0.5, 0.0], potential="none", vparam=[1.0], constraint="none", sigma=0.0,
             dt=1e-3, seed=5, init="box", iparam=[0.0, 50.0], adjacency=adj)
    c.update(kw)
    return c


def test_adj_value_matches_dense(O):
    _, dense = _tiny_graph()
    c = _adj_cfg()
    for i in range(5):
        for j in range(5):
            assert O.adj_value(c, i, j) == dense[i, j]


@pytest.mark.parametrize("i,j", [(0, 1), (0, 2), (1, 3), (2, 4), (1, 2)])
def test_adj_pair_flow_exact(O, i, j):
    """P:1258-1264 is the exact flow of dX^i/dt = alpha (a_ij - beta)(X^j - X^i)
    (P:1252): RK4 of the pair ODE agrees to 1e-10; the midpoint is kept; the
    pair contracts for a_ij > beta and separates for a_ij < beta."""
    _, dense = _tiny_graph()
    c = _adj_cfg()
    alpha, beta, tau = 40.0, 0.5, 1e-3
    xi, xj = np.array([3.0, -1.0]), np.array([-2.0, 4.5])
    yi, yj = O.adj_pair_flow(c, i, j, xi, xj, tau)
    k = alpha * (dense[i, j] - beta)

    def f(u):
        a, b = u[:2], u[2:]
        return np.concatenate([k * (b - a), k * (a - b)])
    u, h = np.concatenate([xi, xj]), tau / 2000
    for _ in range(2000):
        k1 = f(u); k2 = f(u + h / 2 * k1); k3 = f(u + h / 2 * k2); k4 = f(u + h * k3)
        u = u + h / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
    assert np.max(np.abs(np.concatenate([yi, yj]) - u)) < 1e-10
    assert np.allclose(yi + yj, xi + xj, atol=1e-13)
    d0, d1 = np.linalg.norm(xi - xj), np.linalg.norm(yi - yj)
    if dense[i, j] == beta:
        assert abs(d1 - d0) < 1e-12
    else:
        assert (d1 < d0) if dense[i, j] > beta else (d1 > d0)


def test_adj_rbmr_step_conserves_sum(O):
    """Every pair update keeps the pair's sum, so a Jacobi sweep keeps sum_i X^i."""
    c = _adj_cfg()
    x = O.init(c)
    for m in range(20):
        y = O.rbmr_step(c, x, m)
        assert np.allclose(y.sum(0), x.sum(0), rtol=0, atol=1e-10)
        x = y


def test_adj_edge_restricted_slots(O):
    """pairs picked among the nonzeros of A only, uniformly over the
    nnz (directed) entries (chi^2)."""
    adj, dense = _tiny_graph()
    c = _adj_cfg(kparam=[40.0, 0.5, 1.0], n=5)
    nnz = len(adj[1])
    cnt = {}
    for m in range(8000):
        js = O.rbmr_slots(c, m)
        for b in range(len(js) // 2):
            i, j = int(js[2 * b]), int(js[2 * b + 1])
            assert dense[i, j] > 0
            cnt[(i, j)] = cnt.get((i, j), 0) + 1
    obs = np.array(list(cnt.values()), dtype=float)
    assert len(obs) == nnz
    assert stats.chisquare(obs).pvalue > 1e-4


def _mean_field_unstable(adj, n, alpha, beta, k=2):
    """Top-k eigenvectors of the mean-field generator -alpha/(N-1) L_W,
    W_ij = a_ij - beta (i != j): the modes the linear dynamics amplifies."""
    rp, ci, v = adj
    A = np.zeros((n, n))
    A[np.repeat(np.arange(n), np.diff(rp.astype(np.int64))), ci.astype(np.int64)] = v
    W = A - beta
    np.fill_diagonal(W, 0.0)
    L = np.diag(W.sum(1)) - W
    ev, V = np.linalg.eigh(-alpha / (n - 1) * L)
    return ev[-k:], V[:, -k:]


def test_sbm_clusters_recovered_by_oracle(O):
    """The paper's SBM experiment (N = 1200 in blocks 200/400/600,
    p = 0.7, q = 0.3, alpha = 40, beta = 1/2, tau = 1e-3, X_0 ~ U[0, 50]) with
    RBM-r p = 2 to T = 5: (i) each coordinate of the centred positions lies in
    the dominant unstable subspace of the mean-field linear dynamics
    (projection >= 0.85; two nearly degenerate unstable modes, both constant
    on the blocks); (ii) 3-means of the whitened 2-D positions recovers the
    blocks (ARI >= 0.95)."""
    from sklearn.cluster import KMeans
    from sklearn.metrics import adjusted_rand_score
    c = RI.cluster_sbm(seed=3)
    ev, V = _mean_field_unstable(c["adjacency"], 1200, 40.0, 0.5)
    assert ev[0] > 0 and ev[1] > 0
    x = O.run(c, O.init(c), 0, 5000)
    z = x - x.mean(0)
    for a in range(2):
        assert np.linalg.norm(V.T @ z[:, a]) ** 2 / np.dot(z[:, a], z[:, a]) >= 0.85
    w = np.linalg.cholesky(np.linalg.inv(np.cov(z.T)))
    lab = KMeans(3, n_init=10, random_state=0).fit(z @ w).labels_
    assert adjusted_rand_score(c["labels"], lab) >= 0.95
