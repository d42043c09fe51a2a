"""Host-side plumbing of the partitioned single system on CPU (-m "not gpu").

The exchanges between the library's phases (include/rbm.h "Partitioned
single system") move bytes inside the caller-owned workspaces.  Here
DistExchange runs over torch.distributed with the gloo backend, world size
2 and 4, on CPU workspaces laid out by rbm_part_info_get (a host-only call),
and must move exactly the bytes that LoopbackExchange moves when all ranks
live in one process.  No GPU, no kernels: the CUDA side is covered by
tests/test_partition_gpu.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import rbm_inputs as RI

CFG = RI.c5_coulomb_reg(n=60_013, p=8)


def _bufs(G, torch_mod=torch):
    from paper_1812_10575_b200 import partition as PT
    from paper_1812_10575_b200 import rbm as R
    out = []
    for r in range(G):
        info = PT.rbm_part_info_get(R.make_config(dict(CFG, world_size=G, rank=r)))
        g = np.random.default_rng(1000 + r)
        ws = torch_mod.from_numpy(g.integers(0, 256, size=int(info.ws_bytes), dtype=np.uint8))
        out.append(PT.RankBuffers(ws, info))
    return out


def _expected(G, fused=False):
    from paper_1812_10575_b200 import partition as PT
    bufs = _bufs(G)
    ex = PT.LoopbackExchange(fused=fused)
    ex.halo(bufs)
    ex.counts_records(bufs)
    return bufs


def _worker(rank, G, port, q, fused=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    from paper_1812_10575_b200 import partition as PT
    dist.init_process_group("gloo", rank=rank, world_size=G)
    try:
        me = _bufs(G)[rank]
        ex = PT.DistExchange(fused=fused)
        ex.halo([me])
        ex.counts_records([me])
        want = _expected(G, fused)[rank]
        ok = all(torch.equal(a, b) for a, b in zip(me.recv, want.recv))
        ok = ok and torch.equal(me.counts_all, want.counts_all)
        ok = ok and torch.equal(me.halo_recv, want.halo_recv)
        ok = ok and torch.equal(me.ws, want.ws)  # nothing else touched
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("G,fused", [(2, False), (4, False), (2, True)])
def test_dist_exchange_matches_loopback_gloo(G, fused):
    """fused=True: only the counts move (the records were stored in place by
    the kernels); the receive regions must stay untouched."""
    from paper_1812_10575_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, G, port, q, fused)) for r in range(G)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = dict(q.get(timeout=5) for _ in range(G))
    assert all(p.exitcode == 0 for p in procs)
    assert res == {r: True for r in range(G)}


def test_loopback_semantics():
    """Loopback exchange = the documented protocol: chunk j of rank r's send
    array lands in chunk r of rank j's receive array; counts all-gathered
    rank-major; halo of r lands at r+1 (rank 0 receives none)."""
    G = 4
    before = _bufs(G)
    after = _expected(G)
    for r in range(G):
        for j in range(G):
            for a in range(before[0].info.narrays):
                cb = before[0].chunk_bytes[a]
                assert torch.equal(after[j].recv[a][r * cb:(r + 1) * cb], before[r].send[a][j * cb:(j + 1) * cb])
        nb = 4 * before[0].info.nseg
        for s in range(G):
            assert torch.equal(after[r].counts_all[s * nb:(s + 1) * nb], before[s].counts_send)
        if r > 0:
            assert torch.equal(after[r].halo_recv, before[r - 1].halo_send)
        else:
            assert torch.equal(after[0].halo_recv, before[0].halo_recv)
