"""Partitioned single system on one B200 (-m gpu).

All G ranks run in this process on one device with the loopback exchange
(device copies in stream order; no kernel waits on another rank), so every
kernel of the G > 1 path runs exactly as it would with one GPU per rank.

Invariant: the result at any G is bit-identical to G = 1,
because the division is the global (key, id) order and every batch is the
same arithmetic wherever it is computed.  The oracle pins the permutation
(bit-exact) and the one-step states (BASELINE.json tolerances).
"""
import numpy as np
import pytest

import rbm_inputs as RI

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def PT():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1812_10575_b200 import partition, rbm
    rbm.lib()
    return partition


def E(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


def single(cfg, steps):
    from paper_1812_10575_b200 import RBM
    s = RBM(cfg)
    for _ in range(steps):
        s.step()
    out = s.gather(host=False).cpu().numpy()
    s.close()
    return out


def parted(PT, cfg, G, steps):
    ps = PT.PartitionedRBM(cfg, G, range(G), PT.LoopbackExchange())
    ps.run(steps)
    out = ps.gather().cpu().numpy()
    ps.sync()
    ps.close()
    return out


CASES = [
    # (name, cfg): C5-like fp32 d=3 at several p, C4-like, C3-like, fp64 split Dyson,
    # ragged N (N mod p = 1 and >= 2), sphere fp64
    ("c5p2", RI.c5_coulomb_reg(n=200_003, p=2)),
    ("c5p8", RI.c5_coulomb_reg(n=200_003, p=8)),
    ("c5p32", RI.c5_coulomb_reg(n=131_073, p=32)),
    ("c4", RI.c4_aggregation(n=150_001)),
    ("c3", RI.c3_opinion(n=120_000)),
    ("dyson_split", RI.c1_dyson(n=65_536, integrator="split")),
    ("sphere", RI.c2_sphere(n=80_000)),
    ("ragged5", dict(RI.c5_coulomb_reg(n=100_003, p=5), dtype="f64")),
]


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("name,cfg", CASES, ids=[c[0] for c in CASES])
def test_partitioned_bit_identical_to_one_gpu(PT, name, cfg, G):
    if cfg["n"] // G < max(1024, 16 * cfg["p"]):
        pytest.skip("too few particles per rank")
    steps = 5
    a = single(cfg, steps)
    b = parted(PT, cfg, G, steps)
    assert a.shape == b.shape
    assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (
        f"max |diff| {np.max(np.abs(a.astype(np.float64) - b))}")


@pytest.mark.parametrize("G,p", [(2, 2), (4, 3), (8, 8)])
def test_partitioned_permutation_and_step_vs_oracle(PT, O, G, p):
    """Permutation pi_m bit-exact vs the oracle's (key, id) sort, and the
    one-step state within 1e-12 (fp64) of oracle_rbm1_step."""
    cfg = dict(RI.c5_coulomb_reg(n=40_009, p=p), dtype="f64", step0=11)
    ps = PT.PartitionedRBM(cfg, G, range(G), PT.LoopbackExchange())
    x0 = ps.gather().cpu().numpy()
    order = torch.full((cfg["n"],), -1, dtype=torch.int32, device="cuda")
    from paper_1812_10575_b200 import rbm as R
    for s in ps.systems:
        R.rbm_debug_permutation(s.ctx, order.data_ptr())
    ps.step()
    got = order.cpu().numpy().view(np.uint32)
    assert np.array_equal(got, O.permutation(cfg, 11))
    g = ps.gather().cpu().numpy()
    assert E(g, O.rbm1_step(cfg, x0, 11)) <= 1e-12
    ps.close()


def test_partitioned_many_steps_and_user_state(PT):
    """User X_0 (set_state per rank), 40 steps at G=4 == one GPU, bit for bit."""
    from paper_1812_10575_b200 import RBM
    cfg = RI.c4_aggregation(n=90_001)
    x0 = RI.user_x0(cfg["n"], cfg["d"], seed=5).astype(np.float32)
    s = RBM(cfg, x0=x0)
    s.run(40)
    a = s.gather(host=True)
    s.close()
    ps = PT.PartitionedRBM(dict(cfg, init="user"), 4, range(4), PT.LoopbackExchange())
    ps.set_state(x0)
    ps.run(40)
    b = ps.gather().cpu().numpy()
    ps.close()
    assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_partitioned_protocol_errors(PT):
    from paper_1812_10575_b200 import rbm as R
    cfg = dict(RI.c5_coulomb_reg(n=50_000, p=2), world_size=2, rank=0)
    s = R.RBM(cfg)
    with pytest.raises(R.RbmError):
        s.step()                       # rbm_step on a partitioned context
    with pytest.raises(R.RbmError):
        PT.rbm_part_phase1(s.ctx)      # before the prologue
    PT.rbm_part_prologue(s.ctx)
    with pytest.raises(R.RbmError):
        PT.rbm_part_prologue(s.ctx)    # twice
    s.close()


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("name,cfg", [CASES[0], CASES[2], CASES[4], CASES[7]], ids=["c5p2", "c5p32", "c3", "ragged5"])
def test_fused_exchange_bit_identical(PT, name, cfg, G):
    """G9: the bucket step / straddle / prologue store their records straight
    into the destination ranks' receive buffers (double-buffered by step
    parity); the result is bit-identical to one GPU and to the NCCL form."""
    if cfg["n"] // G < max(1024, 16 * cfg["p"]):
        pytest.skip("too few particles per rank")
    steps = 6
    a = single(cfg, steps)
    ps = PT.PartitionedRBM(cfg, G, range(G), PT.LoopbackExchange(fused=True))
    ps.run(steps)
    b = ps.gather().cpu().numpy()
    ps.sync()
    ps.close()
    assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
