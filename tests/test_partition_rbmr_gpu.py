"""RBM-r on one partitioned global system -- -m gpu.

G ranks run in one process on one B200 with the loopback exchange (device
copies in stream order; no kernel waits on another rank).  Rank r owns the ids
[floor(N r/G), floor(N (r+1)/G)) and the batches [floor(nb r/G), ...) of the
sweep; the request / response / increment all-to-alls connect them.  The
state after every step must be bit-identical to the one-GPU RBM-r (reading
D:8: increments summed in ascending global slot order), and the slot draws
bit-exact against the oracle (Algs. 2-3; reading D:9).
"""
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


def cfg_of(kind):
    base = dict(scheme="rbmr", seed=77, step0=3)
    if kind == "smooth_f64_p2":
        return dict(RI.smooth_test(20011, p=2), sigma=0.1, **base)
    if kind == "creg_f32_p8":
        return dict(RI.c5_coulomb_reg(n=50_000, p=8), **base)
    if kind == "dyson_split":
        return dict(RI.c1_dyson(n=10_000, integrator="split"), **base)
    if kind == "sphere":
        return dict(RI.c2_sphere(n=10_000), **base)
    return dict(RI.c4_aggregation(n=40_003), **base)


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("kind", ["smooth_f64_p2", "creg_f32_p8", "dyson_split", "sphere", "c4_p4"])
def test_partitioned_rbmr_bit_identical(R, O, G, kind):
    from paper_1812_10575_b200 import partition as PT
    c = cfg_of(kind)
    one = R.RBM(c)
    x0 = one.gather(host=True)
    ps = PT.PartitionedRBM(c, G, range(G), PT.LoopbackExchange(), device="cuda:0")
    assert all(b.info.phases == 4 and b.info.narrays == 3 for b in ps.bufs)
    for step in range(4):
        one.step()
        ps.step()
        ps.sync()
        got = ps.gather().cpu().numpy()
        ref = one.gather(host=True)
        assert np.array_equal(got, ref), (kind, G, step)
        if step == 0:  # the slots of every rank's batches = the oracle's draws
            slots = np.concatenate([s.slots() for s in ps.systems])
            assert np.array_equal(slots, O.rbmr_slots(c, 3))
            tol = 1e-12 if c["dtype"] == "f64" else 1e-4
            o = O.rbmr_step(c, x0.astype(np.float64), 3)
            assert float(np.max(np.abs(got - o)) / max(1.0, np.max(np.abs(o)))) <= tol
    ps.close()
    one.close()
