"""Partitioned single system across PROCESSES on one B200 (-m gpu), and the
library-communicator parts of the C ABI that one GPU can exercise.

Two processes (gloo process group on 127.0.0.1 for the host-side exchanges)
each drive one rank of a G = 2 system on cuda:0.  With fused=True every rank
maps the other's workspace over CUDA IPC and its bucket / straddle / prologue
kernels store the records straight into the peer's receive buffer -- the
cross-process path that the multi-GPU fused exchange uses over NVLink.  The
exchanges of counts and halo run on host copies after a stream
synchronisation (HostDistExchange), so no kernel ever waits on another rank's
kernel.  The result must be bit-identical to the same global system stepped on
one GPU (world_size 1), SURVEY 8(e) invariant.
"""
import os
import socket

import numpy as np
import pytest

import rbm_inputs as RI

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STEPS = 6


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1812_10575_b200 import rbm
    rbm.lib()
    return rbm


def _cfg(kind):
    if kind == "c5p2":
        return RI.c5_coulomb_reg(n=400_003, p=2)
    if kind == "c4":
        return RI.c4_aggregation(n=300_007)
    return dict(RI.c5_coulomb_reg(n=250_001, p=8), dtype="f64")


def _worker(rank, world, port, kind, fused, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_1812_10575_b200 import partition as PT
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        ps = PT.PartitionedRBM(_cfg(kind), world, [rank], PT.HostDistExchange(fused=fused), device="cuda:0")
        mapped = ps.exchange.fused
        ps.run(STEPS)
        ps.sync()
        ids, x = ps.systems[0].gather_local()
        out = [None] * world
        dist.all_gather_object(out, (ids.cpu().numpy(), x.cpu().numpy(), mapped))
        if rank == 0:
            q.put(out)
        # release the peer mappings on every rank before any rank frees the
        # workspace it exported (CUDA IPC producer/consumer order)
        torch.cuda.synchronize()
        ps.exchange._peer_tensors.clear()
        dist.barrier()
        ps.close()
    except Exception as e:  # report instead of hanging the parent
        if rank == 0:
            q.put(repr(e))
        raise
    finally:
        dist.barrier()
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("kind,fused", [("c5p2", True), ("c4", True), ("f64p8", True), ("c5p2", False)])
def test_two_processes_bit_identical_to_one_gpu(R, kind, fused):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, fused, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=900)
    for p in procs:
        p.join(timeout=120)
    assert not isinstance(got, str), got
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert all(m == fused for _, _, m in got)  # fused: both ranks mapped the peer over CUDA IPC
    ids = np.concatenate([g[0] for g in got]).view(np.uint32)
    xs = np.concatenate([g[1] for g in got])
    c = _cfg(kind)
    n = c["n"]
    assert np.array_equal(np.sort(ids), np.arange(n, dtype=np.uint32))  # every particle once
    x2 = np.empty_like(xs)
    x2[ids] = xs
    one = R.RBM(c)
    one.run(STEPS)
    ref = one.gather(host=True)
    one.close()
    assert np.array_equal(x2, ref)


def test_nccl_unique_id(R):
    a, b = R.rbm_get_nccl_unique_id(), R.rbm_get_nccl_unique_id()
    assert len(a) == 128 and a != b and any(a)


def test_nccl_id_rejected_for_one_gpu(R):
    c = R.make_config(RI.c4_aggregation(n=10_000))
    ws = torch.empty(R.rbm_workspace_size(c), dtype=torch.uint8, device="cuda")
    with pytest.raises(R.RbmError) as e:
        R.rbm_init(c, ws.data_ptr(), ws.numel(), 0, R.rbm_get_nccl_unique_id())
    assert e.value.status == 1


def test_partitioned_without_comm_refuses_rbm_step(R):
    s = R.RBM(dict(RI.c4_aggregation(n=20_000), world_size=2, rank=0))
    with pytest.raises(R.RbmError) as e:
        s.step()
    assert e.value.status == 8
    s.close()


def test_gather_local_one_gpu(R):
    c = RI.c5_coulomb_reg(n=123_457, p=2)
    s = R.RBM(c)
    s.run(3)
    ids, x = s.gather_local()
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), np.arange(c["n"], dtype=np.uint32))
    assert np.array_equal(x.cpu().numpy(), s.gather(host=True))
    s.close()


def test_gather_local_partitioned_loopback(R):
    """Loopback G = 4: the unordered local shards of all ranks hold every
    particle exactly once, with the positions rbm_gather reports."""
    from paper_1812_10575_b200 import partition as PT
    c = RI.c4_aggregation(n=300_007)
    ps = PT.PartitionedRBM(c, 4, range(4), PT.LoopbackExchange(fused=True), device="cuda:0")
    ps.run(3)
    ps.sync()
    full = ps.gather().cpu().numpy()
    ids, xs = [], []
    for s in ps.systems:
        i, x = s.gather_local()
        ids.append(i.cpu().numpy().view(np.uint32))
        xs.append(x.cpu().numpy())
    ids, xs = np.concatenate(ids), np.concatenate(xs)
    assert np.array_equal(np.sort(ids), np.arange(c["n"], dtype=np.uint32))
    assert np.array_equal(xs, full[ids])
    ps.close()
