"""Ensemble mode: replica r on rank r equals the
single-process run with replica = r, bit-exactly.

Two worker processes (world size 2, gloo process group on 127.0.0.1 for the
host-side reduction of their results) each run replica = rank on cuda:0 --
independent systems, no kernel waits on another -- and return a digest of
their final state; the parent runs the same replicas alone and compares.
"""
import hashlib
import os
import socket

import numpy as np
import pytest

import rbm_inputs as RI

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STEPS = 12


def _cfg():
    return RI.c4_aggregation(n=300_007)


def _digest(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_1812_10575_b200.ensemble import run_replica
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    x = run_replica(_cfg(), rank, STEPS)
    out = [None] * world
    dist.all_gather_object(out, (rank, _digest(x), float(np.mean(x[:, 0]))))
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_ensemble_replica_r_equals_single_run():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    from paper_1812_10575_b200.ensemble import run_replica
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    single = {r: _digest(run_replica(_cfg(), r, STEPS)) for r in range(2)}
    assert {r: d for r, d, _ in got} == single
    assert single[0] != single[1]
