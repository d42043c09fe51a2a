"""Partitioned single system over G ranks.

The production path is CommPartitionedRBM: rbm_init receives an NCCL id and
librbm.so runs the whole step -- kernels and NCCL exchanges, captured into
CUDA graphs -- on one process per GPU; torch.distributed only broadcasts the
id.  The rest of this module drives the caller-exchange protocol of the same
library (rbm_part_* phases), used to test the G > 1 kernels without several
GPUs.  The step's three exchanges:

    H  halo     rank r's halo_send -> rank r+1's halo_recv (<= p-1 records)
    C  counts   all-gather of counts_send (2^b1 u32 per rank) -> counts_all
    R  records  all-to-all, equal chunks, of the state records

Protocol per context: rbm_init; prologue; C; R; then per step
phase1; H; phase2; C; R.

Interchangeable caller exchanges move the bytes, on byte views of the
caller-owned workspaces (offsets from rbm_part_info_get):

  DistExchange      one rank per process, torch.distributed (NCCL over
                    NVLink on B200; gloo for the CPU tests of this plumbing)
  HostDistExchange  the same with the collectives on host copies (gloo with
                    device workspaces): several processes on ONE device
  LoopbackExchange  all G ranks in one process on one device: plain device
                    copies, run in stream order (no kernel waits on another
                    rank), used to test the G > 1 kernels on one GPU

fused=True (either exchange, G <= 8): the kernels store the records straight
into the destination rank's receive buffer (peer memory over NVLink, mapped
with CUDA IPC by DistExchange) and exchange R disappears.
"""
from __future__ import annotations

import ctypes as C

from . import rbm as R


class RbmPartInfo(C.Structure):
    _fields_ = [
        ("ws_bytes", C.c_uint64), ("world_size", C.c_uint32), ("rank", C.c_uint32),
        ("nseg", C.c_uint32), ("narrays", C.c_uint32), ("chunk_elems", C.c_uint64),
        ("send_off", C.c_uint64 * 5), ("recv_off", C.c_uint64 * 5), ("elem_bytes", C.c_uint32 * 5),
        ("counts_send_off", C.c_uint64), ("counts_all_off", C.c_uint64),
        ("halo_send_off", C.c_uint64), ("halo_recv_off", C.c_uint64), ("halo_bytes", C.c_uint64),
        ("id0", C.c_uint64), ("n0", C.c_uint64),
        ("chunk_bytes", C.c_uint64 * 5), ("phases", C.c_uint32), ("pad", C.c_uint32),
    ]


_sig_done = False


def _lib():
    global _sig_done
    L = R.lib()
    if not _sig_done:
        L.rbm_part_info_get.restype = C.c_int
        L.rbm_part_info_get.argtypes = [C.POINTER(R.RbmConfig), C.POINTER(RbmPartInfo)]
        for name in ("rbm_part_prologue", "rbm_part_phase1", "rbm_part_phase2"):
            f = getattr(L, name)
            f.restype, f.argtypes = C.c_int, [C.c_void_p]
        L.rbm_part_set_peers.restype = C.c_int
        L.rbm_part_set_peers.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.c_uint32]
        L.rbm_part_phase.restype = C.c_int
        L.rbm_part_phase.argtypes = [C.c_void_p, C.c_uint32]
        _sig_done = True
    return L


def rbm_part_info_get(cfg: R.RbmConfig) -> RbmPartInfo:
    out = RbmPartInfo()
    R._check(_lib().rbm_part_info_get(C.byref(cfg), C.byref(out)))
    return out


def rbm_part_set_peers(ctx, peer_ws_ptrs):
    arr = (C.c_uint64 * len(peer_ws_ptrs))(*[int(p) for p in peer_ws_ptrs])
    R._check(_lib().rbm_part_set_peers(ctx, arr, len(peer_ws_ptrs)), ctx)


def rbm_part_prologue(ctx):
    R._check(_lib().rbm_part_prologue(ctx), ctx)


def rbm_part_phase1(ctx):
    R._check(_lib().rbm_part_phase1(ctx), ctx)


def rbm_part_phase2(ctx):
    R._check(_lib().rbm_part_phase2(ctx), ctx)


def rbm_part_phase(ctx, k: int):
    R._check(_lib().rbm_part_phase(ctx, int(k)), ctx)


class RankBuffers:
    """Byte views of one rank's exchanged regions inside its workspace tensor."""

    def __init__(self, ws, info: RbmPartInfo):
        self.ws, self.info = ws, info
        G = info.world_size

        def v(off, nbytes):
            return ws[off:off + nbytes]

        self.chunk_bytes = [int(info.chunk_bytes[a]) for a in range(info.narrays)]
        self.send = [v(info.send_off[a], G * self.chunk_bytes[a]) for a in range(info.narrays)]
        self.recv = [v(info.recv_off[a], G * self.chunk_bytes[a]) for a in range(info.narrays)]
        self.counts_send = v(info.counts_send_off, 4 * info.nseg)
        self.counts_all = v(info.counts_all_off, 4 * info.nseg * G)
        self.halo_send = v(info.halo_send_off, info.halo_bytes)
        self.halo_recv = v(info.halo_recv_off, info.halo_bytes)

    @property
    def rank(self) -> int:
        return int(self.info.rank)


class LoopbackExchange:
    """All G ranks in this process (one device): exchanges are device copies.
    With fused=True the records are already in place (the kernels stored them
    into the peers' receive buffers); only the counts are gathered."""

    def __init__(self, fused: bool = False):
        self.fused = fused

    def peers(self, ranks):
        """Workspace base of every rank, as usable from this device."""
        return [b.ws.data_ptr() for b in ranks]

    def counts_records(self, ranks):
        G = len(ranks)
        nb = 4 * ranks[0].info.nseg
        for dst in ranks:
            for s, src in enumerate(ranks):
                dst.counts_all[s * nb:(s + 1) * nb].copy_(src.counts_send)
        if self.fused:
            return
        for a in range(ranks[0].info.narrays):
            cb = ranks[0].chunk_bytes[a]
            for r, src in enumerate(ranks):
                for j in range(G):
                    ranks[j].recv[a][r * cb:(r + 1) * cb].copy_(src.send[a][j * cb:(j + 1) * cb])

    def halo(self, ranks):
        for r in range(len(ranks) - 1):
            ranks[r + 1].halo_recv.copy_(ranks[r].halo_send)

    def alltoall(self, ranks, a):
        """All-to-all of equal chunks of exchanged array a (RBM-r exchanges)."""
        G = len(ranks)
        cb = ranks[0].chunk_bytes[a]
        for r, src in enumerate(ranks):
            for j in range(G):
                ranks[j].recv[a][r * cb:(r + 1) * cb].copy_(src.send[a][j * cb:(j + 1) * cb])


class DistExchange:
    """One rank per process over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None, fused: bool = False):
        import torch.distributed as dist
        self.dist, self.group, self.fused = dist, group, fused
        self._peer_tensors = []

    def peers(self, ranks):
        """Fused mode: map every rank's workspace into this process (CUDA IPC,
        peer access over NVLink) and return the base pointers."""
        from torch.multiprocessing.reductions import reduce_tensor
        (me,) = ranks
        G = int(me.info.world_size)
        fn, args = reduce_tensor(me.ws)
        allh = [None] * G
        self.dist.all_gather_object(allh, (fn, args), group=self.group)
        ptrs = []
        for j, (f, a) in enumerate(allh):
            if j == me.rank:
                ptrs.append(me.ws.data_ptr())
            else:
                t = f(*a)
                self._peer_tensors.append(t)
                ptrs.append(t.data_ptr())
        return ptrs

    def counts_records(self, ranks):
        (me,) = ranks
        d = self.dist
        d.all_gather_into_tensor(me.counts_all, me.counts_send, group=self.group)
        if self.fused:
            return
        for a in range(me.info.narrays):
            d.all_to_all_single(me.recv[a], me.send[a], group=self.group)

    def alltoall(self, ranks, a):
        (me,) = ranks
        self.dist.all_to_all_single(me.recv[a], me.send[a], group=self.group)

    def halo(self, ranks):
        (me,) = ranks
        d, r, G = self.dist, me.rank, int(me.info.world_size)
        ops = []
        if r + 1 < G:
            ops.append(d.P2POp(d.isend, me.halo_send, r + 1, group=self.group))
        if r > 0:
            ops.append(d.P2POp(d.irecv, me.halo_recv, r - 1, group=self.group))
        if ops:
            for q in d.batch_isend_irecv(ops):
                q.wait()


class HostDistExchange(DistExchange):
    """DistExchange whose collectives run on host copies (gloo with device
    workspaces): the counts and the halo are staged through CPU tensors, so
    every exchange is preceded by a stream synchronisation of this rank.  Used
    to run the fused path's cross-process CUDA-IPC stores with several ranks
    on ONE device (tests): no kernel ever waits on another rank's kernel."""

    def counts_records(self, ranks):
        (me,) = ranks
        d = self.dist
        G = int(me.info.world_size)
        cs = me.counts_send.cpu()
        out = [self.torch.empty_like(cs) for _ in range(G)]
        d.all_gather(out, cs, group=self.group)
        me.counts_all.copy_(self.torch.cat(out).to(me.counts_all.device))
        if self.fused:
            return
        for a in range(me.info.narrays):  # gloo has no all-to-all: all-gather, keep chunk `rank`
            cb = me.chunk_bytes[a]
            send = me.send[a].cpu()
            allv = [self.torch.empty_like(send) for _ in range(G)]
            d.all_gather(allv, send, group=self.group)
            r = me.rank
            me.recv[a].copy_(self.torch.cat([v[r * cb:(r + 1) * cb] for v in allv]).to(me.recv[a].device))

    def halo(self, ranks):
        (me,) = ranks
        d, r, G = self.dist, me.rank, int(me.info.world_size)
        if r + 1 < G:
            d.send(me.halo_send.cpu(), r + 1, group=self.group)
        if r > 0:
            buf = self.torch.empty(me.halo_recv.numel(), dtype=me.halo_recv.dtype)
            d.recv(buf, r - 1, group=self.group)
            me.halo_recv.copy_(buf.to(me.halo_recv.device))

    def alltoall(self, ranks, a):  # gloo has no all-to-all: all-gather, keep chunk `rank`
        (me,) = ranks
        G, r, cb = int(me.info.world_size), me.rank, me.chunk_bytes[a]
        send = me.send[a].cpu()
        allv = [self.torch.empty_like(send) for _ in range(G)]
        self.dist.all_gather(allv, send, group=self.group)
        me.recv[a].copy_(self.torch.cat([v[r * cb:(r + 1) * cb] for v in allv]).to(me.recv[a].device))

    @property
    def torch(self):
        import torch
        return torch


class CommPartitionedRBM:
    """One rank of a global RBM-1 system whose whole step -- kernels and the
    NCCL exchanges -- runs inside librbm.so (rbm_init with an NCCL id; rbm_run
    replays CUDA graphs of steps with their NCCL calls).  torch.distributed
    only broadcasts the 128-byte id (plumbing).  fused=True maps the peers'
    workspaces over CUDA IPC in the library (rbm_part_map_peers) so the bucket
    step stores the records straight into their destination ranks; the NCCL
    all-to-all is used if any rank cannot map."""

    def __init__(self, cfg: dict, world_size: int, rank: int, device=None, fused: bool = True, group=None):
        import torch.distributed as dist
        obj = [R.rbm_get_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        self.cfg = dict(cfg, world_size=int(world_size), rank=int(rank))
        self.system = R.RBM(self.cfg, device=device, nccl_id=obj[0])
        self.fused = False
        if fused and world_size <= 8:
            try:
                R.rbm_part_map_peers(self.system.ctx)
                self.fused = True
            except R.RbmError:
                self.fused = False

    def run(self, nsteps: int):
        self.system.run(nsteps)

    def step(self):
        self.system.step()

    def sync(self):
        self.system.sync()

    def gather(self, host: bool = False):
        """Whole state in id order on every rank (collective)."""
        return self.system.gather(host=host)

    def gather_local(self):
        return self.system.gather_local()

    @property
    def stream(self):
        return self.system.stream

    @property
    def launches_per_step(self) -> int:
        return self.system.launches_per_step

    def close(self):
        self.system.close()


class PartitionedRBM:
    """One global RBM-1 system split over `world_size` ranks.

    `ranks`: the ranks this process drives (all of them for the loopback
    exchange on one device; [rank] under torch.distributed)."""

    def __init__(self, cfg: dict, world_size: int, ranks, exchange, device=None):
        import torch
        self.torch = torch
        self.cfg, self.G, self.exchange = dict(cfg), int(world_size), exchange
        self.systems, self.bufs = [], []
        for r in ranks:
            c = dict(self.cfg, world_size=self.G, rank=int(r))
            s = R.RBM(c, device=device)
            info = rbm_part_info_get(s.c)
            assert info.ws_bytes == s.ws_bytes
            self.systems.append(s)
            self.bufs.append(RankBuffers(s.ws, info))
        if getattr(exchange, "fused", False):
            exchange.fused = False
            if not self.enable_fused():
                raise RuntimeError("fused exchange: peer workspaces could not be mapped on every rank")
        self.n, self.d = int(self.cfg["n"]), int(self.cfg["d"])
        self.dtype = self.systems[0].dtype
        self.device = self.systems[0].device
        self.started = False

    def enable_fused(self) -> bool:
        """Map every rank's workspace (collective under torch.distributed) and
        switch the kernels to storing records straight into the peers'
        receive buffers.  All ranks agree; on any failure none switches."""
        torch = self.torch
        ok, ptrs = 1, None
        try:
            ptrs = self.exchange.peers(self.bufs)
        except Exception:
            ok = 0
        if isinstance(self.exchange, DistExchange):
            cpu = isinstance(self.exchange, HostDistExchange)
            t = torch.tensor([ok], dtype=torch.int32, device="cpu" if cpu else self.device)
            self.exchange.dist.all_reduce(t, op=self.exchange.dist.ReduceOp.MIN, group=self.exchange.group)
            ok = int(t.item())
        if ok:
            for s in self.systems:
                rbm_part_set_peers(s.ctx, ptrs)
            self.exchange.fused = True
        return bool(ok)

    def set_state(self, x_full):
        """X_0 in id order (N x d, host array or device tensor): each rank takes its ids."""
        for s, b in zip(self.systems, self.bufs):
            i0, n0 = int(b.info.id0), int(b.info.n0)
            s.set_state(x_full[i0:i0 + n0])
        self.started = False

    def _start(self):
        for s in self.systems:
            rbm_part_prologue(s.ctx)
        self.exchange.counts_records(self.bufs)
        self.started = True

    def step(self):
        if self.bufs[0].info.phases == 4:  # RBM-r: request, response, increment exchanges
            for k in range(1, 5):
                for s in self.systems:
                    rbm_part_phase(s.ctx, k)
                if k < 4:
                    self.exchange.alltoall(self.bufs, k - 1)
            return
        if not self.started:
            self._start()
        for s in self.systems:
            rbm_part_phase1(s.ctx)
        self.exchange.halo(self.bufs)
        for s in self.systems:
            rbm_part_phase2(s.ctx)
        self.exchange.counts_records(self.bufs)

    def run(self, nsteps: int):
        for _ in range(int(nsteps)):
            self.step()

    def gather_local(self, out=None):
        """Device tensor (N x d): rows of the ids held by this process's ranks
        (other rows zero)."""
        torch = self.torch
        if out is None:
            out = torch.zeros((self.n, self.d), dtype=self.dtype, device=self.device)
        for s in self.systems:
            R.rbm_gather(s.ctx, 0, self.n, out.data_ptr(), R.MEM_DEVICE)
        return out

    def gather(self, group=None):
        """Full state in id order on every process (device tensor).  Under
        torch.distributed the disjoint per-rank rows are combined by an
        integer SUM over the bit patterns (exact: every other rank adds 0)."""
        out = self.gather_local()
        if not isinstance(self.exchange, DistExchange):
            return out
        torch = self.torch
        iv = out.view(torch.int64 if self.dtype == torch.float64 else torch.int32)
        self.exchange.dist.all_reduce(iv, group=group)
        return out

    def sync(self):
        for s in self.systems:
            s.sync()

    @property
    def step_index(self) -> int:
        return self.systems[0].step_index

    def close(self):
        for s in self.systems:
            s.close()
