"""Seeded synthetic workloads shared by tests/ and bench.py.

Holds NONE of the method's arithmetic: only the BASELINE.json configurations
(C1..C5) as plain dicts, and seeded numpy arrays for user-supplied initial
data (RBM_INIT_USER).  Both the oracle shim (oracle/oracle.py) and the product
binding (paper_1812_10575_b200/rbm.py) accept these dicts.

Keys: d, n, p, dtype ('f32'|'f64'), scheme ('rbm1'|'rbmr'), integrator
('em'|'split'), kernel, kparam, potential ('none'|'harmonic'), vparam,
constraint ('none'|'sphere'), sigma, dt, seed, replica, init, iparam, steps.
"""
from __future__ import annotations

import math

import numpy as np


def c1_dyson(n: int = 500, integrator: str = "em", scheme: str = "rbm1", seed: int = 1) -> dict:
    """BASELINE.json configs[0]: Dyson Brownian motion."""
    return dict(d=1, n=n, p=2, dtype="f64", scheme=scheme, integrator=integrator,
                kernel="dyson", kparam=[], potential="harmonic", vparam=[1.0],
                constraint="none", sigma=math.sqrt(2.0 / (n - 1)), dt=1e-3, seed=seed,
                init="normal", iparam=[0.0, 1.0], steps=1000)


def c2_sphere(n: int = 10**6, seed: int = 1, scheme: str = "rbm1") -> dict:
    """BASELINE.json configs[1]: Thomson-type Coulomb on S^2."""
    return dict(d=3, n=n, p=2, dtype="f64", scheme=scheme, integrator="em",
                kernel="coulomb", kparam=[], potential="none", vparam=[1.0],
                constraint="sphere", sigma=0.0, dt=1e-4, seed=seed,
                init="sphere", iparam=[], steps=200)


def c3_opinion(n: int = 10**7, seed: int = 1, scheme: str = "rbm1") -> dict:
    """BASELINE.json configs[2]: bounded-confidence opinion."""
    return dict(d=1, n=n, p=2, dtype="f32", scheme=scheme, integrator="em",
                kernel="bounded_confidence", kparam=[1.0, 1.0], potential="none",
                vparam=[1.0], constraint="none", sigma=0.01, dt=1e-2, seed=seed,
                init="box", iparam=[-5.0, 5.0], steps=500)


def opinion_paper(n: int = 1000, noise: bool = False, seed: int = 1, dtype: str = "f64") -> dict:
    """The paper's stochastic opinion dynamics: alpha = 40,
    closed window phi = chi_[0,1], tau = 1e-4, N = 1e3, eps_N = 0 or N^{-1/3}.
    The paper does not state the initial data; U[-5, 5] as in C3 (D:25)."""
    return dict(d=1, n=n, p=2, dtype=dtype, scheme="rbm1", integrator="em",
                kernel="bounded_confidence", kparam=[40.0, 1.0, 1.0], potential="none",
                vparam=[1.0], constraint="none", sigma=(n ** (-1.0 / 3.0)) if noise else 0.0,
                dt=1e-4, seed=seed, init="box", iparam=[-5.0, 5.0], steps=10000)


def c4_aggregation(n: int = 10**8, seed: int = 1, scheme: str = "rbm1") -> dict:
    """BASELINE.json configs[3]: 2-D Gaussian attraction-repulsion (synthetic)."""
    return dict(d=2, n=n, p=4, dtype="f32", scheme=scheme, integrator="em",
                kernel="gauss_attr_rep", kparam=[], potential="harmonic", vparam=[1.0],
                constraint="none", sigma=0.05, dt=5e-3, seed=seed,
                init="mixture", iparam=[5, 0.5, -4.0, 4.0], steps=100)


def c5_coulomb_reg(n: int = 2**28, p: int = 2, seed: int = 1, scheme: str = "rbm1") -> dict:
    """BASELINE.json configs[4]: 3-D regularised Coulomb, 2^28 particles per GPU."""
    return dict(d=3, n=n, p=p, dtype="f32", scheme=scheme, integrator="em",
                kernel="coulomb_reg", kparam=[0.01], potential="harmonic", vparam=[1.0],
                constraint="none", sigma=0.1, dt=1e-3, seed=seed,
                init="normal", iparam=[0.0, 1.0], steps=50)


def smooth_test(n: int, p: int = 2, beta: float = 1.0, dtype: str = "f64", seed: int = 1) -> dict:
    """The paper's smooth test system K(z)=z/(1+z^2), V=beta x^2/2."""
    return dict(d=1, n=n, p=p, dtype=dtype, scheme="rbm1", integrator="em",
                kernel="smooth", kparam=[], potential="harmonic" if beta else "none",
                vparam=[beta], constraint="none", sigma=0.0, dt=2.0**-7, seed=seed,
                init="normal", iparam=[0.0, 1.0], steps=128)


def wealth(n: int = 10**5, integrator: str = "split", seed: int = 1, kappa: float = 1.0,
           diff: float = 1.0, dtype: str = "f64") -> dict:
    """Wealth model (Sec. 5.2.1): dY = -kappa (Y - Y_theta) dt +
    sqrt(2D) Y dB (quadratic trading phi = y^2/2, multiplicative noise), RBM-1
    with p = 2 solved by splitting; X_0 = |N(0,1)|; tau = 1e-3, T = 3."""
    return dict(d=1, n=n, p=2, dtype=dtype, scheme="rbm1", integrator=integrator,
                kernel="linear", kparam=[kappa], potential="none", vparam=[1.0],
                constraint="none", noise="geometric", sigma=math.sqrt(2.0 * diff), dt=1e-3,
                seed=seed, init="abs_normal", iparam=[0.0, 1.0], steps=3000)


def second_order(n: int = 2**24, p: int = 2, seed: int = 1, scheme: str = "rbm1") -> dict:
    """The paper's second-order system at scale: X' = V, V' = mean
    over the batch of K(X^i - X^j) - beta X^i with the smooth test kernel,
    position Verlet with the paper's start step, fp64, stored as d = 2
    components (x, v) at the start and (x_n, x_{n-1}) after; (x_0, v_0) iid
    N(0, 1) (the paper's example size is N = 500; this is the same system at
    2^24 particles for the throughput line)."""
    return dict(d=2, n=n, p=p, dtype="f64", scheme=scheme, integrator="verlet", kernel="smooth",
                kparam=[], potential="harmonic", vparam=[1.0], constraint="none", sigma=0.0,
                dt=2.0 ** -7, seed=seed, init="normal", iparam=[0.0, 1.0], state_form="xv", steps=100)


def sbm_adjacency(sizes=(200, 400, 600), p_in: float = 0.7, q_out: float = 0.3, seed: int = 1):
    """Stochastic block model: symmetric 0/1 adjacency,
    P(a_ij = 1) = p_in inside a block, q_out across, no self loops; CSR with
    rows sorted by column: (row_ptr u32, col u32, val f64), plus the labels."""
    rng = np.random.default_rng(seed)
    n = int(sum(sizes))
    lab = np.repeat(np.arange(len(sizes)), sizes)
    prob = np.where(lab[:, None] == lab[None, :], p_in, q_out)
    up = np.triu(rng.random((n, n)) < prob, 1)
    a = up | up.T
    rows, cols = np.nonzero(a)
    rp = np.zeros(n + 1, dtype=np.uint32)
    np.cumsum(np.bincount(rows, minlength=n), out=rp[1:])
    return (rp, cols.astype(np.uint32), np.ones(len(cols))), lab


def cluster_sbm(d: int = 2, seed: int = 1, graph_seed: int = 1, edge_restricted: bool = False,
                scheme: str = "rbmr", dtype: str = "f64") -> dict:
    """Clustering through the particle system (Sec. 5.3): SBM with
    N = 1200 (200/400/600, p = 0.7, q = 0.3), alpha = 40, beta = 1/2,
    tau = 1e-3, X_0 ~ U[0, 50]^d, RBM-r with p = 2 and the exact pair update
    (P:1258-1264); one step = N/2 pair picks = tau.  d = 2 (reading
    D:26): each coordinate follows the paper's dynamics with the same picks."""
    adj, lab = sbm_adjacency(seed=graph_seed)
    return dict(d=d, n=1200, p=2, dtype=dtype, scheme=scheme, integrator="split", kernel="adjacency",
                kparam=[40.0, 0.5, 1.0 if edge_restricted else 0.0], potential="none", vparam=[1.0],
                constraint="none", sigma=0.0, dt=1e-3, seed=seed, init="box", iparam=[0.0, 50.0],
                adjacency=adj, labels=lab, steps=5000)


ALL = {"C1": c1_dyson, "C2": c2_sphere, "C3": c3_opinion, "C4": c4_aggregation, "C5": c5_coulomb_reg,
       "verlet": second_order}


def user_x0(n: int, d: int, seed: int, dist: str = "normal", scale: float = 1.0) -> np.ndarray:
    """Seeded user initial data in id order, shape (n, d), float64."""
    rng = np.random.default_rng(seed)
    if dist == "normal":
        return scale * rng.standard_normal((n, d))
    if dist == "uniform":
        return scale * rng.uniform(-1.0, 1.0, (n, d))
    if dist == "sphere":
        z = rng.standard_normal((n, d))
        return z / np.linalg.norm(z, axis=1, keepdims=True)
    raise ValueError(dist)


def semicircle_x0(n: int, seed: int, radius: float = 2.0) -> np.ndarray:
    """Seeded iid sample of rho_0(x) = sqrt(R^2 - x^2) / (pi R^2 / 2) on [-R, R]
    (PAPER.md:823-825 with R = 2; the paper draws it by Metropolis-Hastings,
    here by exact rejection sampling), shape (n, 1)."""
    rng = np.random.default_rng(seed)
    out = np.empty(0)
    while out.size < n:
        x = rng.uniform(-radius, radius, 2 * n)
        keep = rng.uniform(0.0, 1.0, 2 * n) < np.sqrt(np.maximum(radius * radius - x * x, 0.0)) / radius
        out = np.concatenate([out, x[keep]])
    return out[:n].reshape(n, 1)

