#!/usr/bin/env python
"""RBM time-step benchmark (BASELINE.json metric: particle-steps/s + HBM GB/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5] [--p 2]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference          # the CPU oracle arm

A "step" is one RBM-1 time step (Alg. 1) of the whole
workload: fresh random division, intra-batch interactions, Euler-Maruyama
update.  Default workload: BASELINE.json configs[4] (C5), 2^28 particles per
GPU, fp32, d=3, regularised Coulomb, p=2.  At N>1 GPUs (torchrun) the default
is C5's partitioned single system: one global system of N x 2^28 particles
split by key range over the ranks, exchanges over NCCL (weak scaling);
--mode ensemble runs independent replicas instead (replica = rank).

Timing: W untimed warm-up steps, then exactly K steps (rbm_run, the user API,
CUDA-graph replays) bracketed by a barrier and torch.cuda.synchronize() on
both sides, measured with CUDA events on the library's stream, max over
ranks.  The state (4-5 GB at C5) is larger than the 126 MB L2, so no flush is
needed between steps.  Per-kernel device times come from a second window of K
eager steps in which the library records CUDA events around its kernels
(rbm_timing_begin/end); roofline.frac uses SURVEY 8(d)'s algorithmic bytes
(2 d s per particle-step) over the dominant kernel's mean launch time.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import rbm_inputs as RI  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C5", choices=["C1", "C2", "C3", "C4", "C5", "wealth", "verlet", "opinion"])
    ap.add_argument("--p", type=int, default=None, help="batch size override (C5: 2, 8, 32)")
    ap.add_argument("--scheme", default="rbm1", choices=["rbm1", "rbmr", "rbmr_seq"])
    ap.add_argument("--n", type=int, default=None, help="particles per GPU override")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="fused", choices=["fused", "nccl", "torch"],
                    help="partitioned mode: the library's NCCL exchanges with records stored into the "
                         "peers' buffers by the kernels (fused, CUDA IPC) or moved by an NCCL all-to-all "
                         "(nccl); torch: the caller-exchange protocol over torch.distributed")
    ap.add_argument("--direct", action="store_true",
                    help="time the direct O(N^2) step (row f1) on the workload's model instead")
    ap.add_argument("--mode", default=None, choices=["partition", "ensemble"],
                    help="N>1 GPUs: one partitioned global system (default) or independent replicas")
    return ap.parse_args()


def workload(args, rank: int) -> dict:
    kw = {"scheme": args.scheme}
    if args.n:
        kw["n"] = args.n
    if args.workload == "C5":
        cfg = RI.c5_coulomb_reg(p=args.p or 2, **kw)
    elif args.workload == "wealth":
        cfg = RI.wealth(**{k: v for k, v in kw.items() if k != "scheme"})
    elif args.workload == "opinion":  # the paper's opinion dynamics with eps_N noise (row f4)
        cfg = RI.opinion_paper(noise=True, **{k: v for k, v in kw.items() if k != "scheme"})
    else:
        cfg = RI.ALL[args.workload](**kw)
        if args.p:
            cfg["p"] = args.p
    cfg["replica"] = rank
    return cfg


def elt(cfg):
    return 8 if cfg["dtype"] == "f64" else 4


def rec_bytes(cfg):
    """Bytes of one state record {id, [key,] x} (RecL in csrc/rbm_device.cuh)."""
    raw = 4 + cfg["d"] * elt(cfg)
    if raw <= 8:
        return 8
    if raw <= 16:
        return 16
    return 24 if (elt(cfg) == 8 and raw + 4 <= 24) else 32


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            P = json.load(f)
        return float(P["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def alg_bytes(name: str, cfg: dict) -> float:
    """ALGORITHMIC HBM bytes per launch: the method reads and
    writes each particle's state once per step, 2 d s bytes per particle-step
    (s = bytes per scalar).  Only the kernel that performs the step's update
    (the bucket step / resident step / RBM-r apply) is credited with them; ids,
    shuffle keys and the permutation moves are the overhead of realising a
    random division on a bandwidth machine (8(d) "Algorithmic bytes")."""
    per = 2.0 * cfg["d"] * elt(cfg) * cfg["n"]
    # RBM-r: the emit kernel reads x_{j_s} once per slot (d s per particle-step,
    # random sectors), the apply kernel reads and writes each position;
    # RBM-r': the sweep reads and writes the members' positions (random)
    return {"bucket_step": per, "rbmr_apply": per, "rbmr_emit": per / 2,
            "rbmr_seq_sweep": per}.get(name, 0.0)


def design_bytes(name: str, cfg: dict, layout) -> float:
    """Bytes per launch THIS design must move: one read
    and one write of the RS-byte state record per particle, plus the 4-byte
    side key pass 2 writes and the bucket step reads when the record has no
    room for it (2-pass layouts).  Reported beside the algorithmic figure so
    that traffic-inflating designs cannot hide (8(d) "useful GB/s")."""
    n = cfg["n"]
    R = rec_bytes(cfg)
    keyed = 8 + cfg["d"] * elt(cfg) <= R
    side = 4.0 if (not keyed and layout[1] == 2) else 0.0
    rbmr = n * (4 * elt(cfg) + 4 * elt(cfg) + 4 + 4 + 8)
    return {"split": (2.0 * R + side) * n, "bucket_step": (2.0 * R + side) * n,
            "rbmr_batch": float(rbmr)}.get(name, 0.0)


class Clocks:
    """nvidia-smi sampler running during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def stop(self):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 6 and r[0].isdigit()]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = sorted(int(r[0]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[2 + k].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": int(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


def cpu_baseline(cfg: dict, budget_s: float = 12.0, n_sample: int = 1 << 19) -> dict:
    """The oracle as it stands, single-threaded, on a bounded sample of the
    same workload (same config, N = n_sample particles)."""
    import numpy as np

    from oracle import oracle as O
    c = dict(cfg, n=min(cfg["n"], n_sample))
    x = O.init(c)
    t0 = time.perf_counter()
    x = O.rbm1_step(c, x, 0) if c["scheme"] == "rbm1" else O.rbmr_step(c, x, 0)
    t1 = time.perf_counter() - t0
    k = int(max(1, min(40, budget_s / max(t1, 1e-6))))
    t0 = time.perf_counter()
    x = O.run(c, x, 1, k)
    dt = time.perf_counter() - t0
    assert np.isfinite(x).all()
    return {"value": c["n"] * k / dt, "unit": "particle-steps/s", "cores": 1, "kind": "oracle",
            "sample": f"{c['n']} particles of the same workload, {k} steps (oracle is single-threaded; host nproc={os.cpu_count()})"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = workload(args, 0)
    from oracle import oracle as O
    c = dict(cfg, n=min(cfg["n"], 1 << 17))
    x = O.init(c)
    x = O.run(c, x, 0, args.warmup)
    t0 = time.perf_counter()
    x = O.run(c, x, args.warmup, args.steps)
    dt = time.perf_counter() - t0
    v = c["n"] * args.steps / dt
    line = {"impl": "reference", "metric": "particle-steps/s", "value": v, "unit": "particle-steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(config_dict(args, c, args.gpus), sample_of=f"{args.workload} at n_per_gpu={cfg['n']}"),
            "cpu_baseline": {"value": v, "unit": "particle-steps/s", "cores": 1, "kind": "oracle",
                             "sample": f"{c['n']} particles of the workload per step (oracle, 1 thread)"},
            "e2e": {"value": v, "unit": "particle-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def config_dict(args, cfg, world):
    return {"workload": f"{args.workload} " + {
        "C1": "Dyson Brownian motion", "C2": "Thomson-type Coulomb on S^2",
        "C3": "bounded-confidence opinion", "C4": "2-D Gaussian aggregation",
        "C5": "3-D regularised Coulomb, partitioned-system size per GPU",
        "wealth": "wealth model (paper Sec. 5.2.1, row f4)",
        "verlet": "second-order system, position Verlet (paper Sec. 4.3, row f3)",
        "opinion": "opinion dynamics, closed window, eps_N noise (paper Sec. 5.2.2, row f4)"}[args.workload],
        "n_per_gpu": cfg["n"], "d": cfg["d"], "p": cfg["p"], "scheme": cfg["scheme"],
        "kernel": cfg["kernel"], "integrator": cfg["integrator"], "dt": cfg["dt"],
        "sigma": cfg["sigma"],
        "multi_gpu": "single system" if world == 1 else "ensemble replicas (replica = rank), no collective",
        "l2": "inputs larger than L2 (state >> 126 MB); no flush"
        if cfg["n"] * (4 + cfg["d"] * elt(cfg)) > 2 * 126e6 else "state fits in L2; no flush"}


def direct_peak(cfg):
    """ALU roofline of one fp32/fp64 interaction on B200:
    148 SMs x 1.965 GHz x (128 fp32 | 64 fp64 FMA-pipe lanes per SM per clock)
    / (pipe instructions per interaction), and the MUFU bound (16/clk/SM)."""
    lanes = 64.0 if cfg["dtype"] == "f64" else 128.0
    instr = {"coulomb_reg": 12, "smooth": 10, "gauss_attr_rep": 14, "bounded_confidence": 8,
             "dyson": 6, "coulomb": 12, "zero": 4}[cfg["kernel"]] + 2 * cfg["d"]
    return 148 * 1.965e9 * lanes / instr


def bench_direct(args, cfg, dev, local):
    """Row f1: fully coupled Euler-Maruyama steps, interactions per second."""
    import numpy as np
    import torch

    from paper_1812_10575_b200 import Direct
    n = args.n or (1 << 16)
    c = dict(cfg, n=n)
    x0 = RI.user_x0(n, c["d"], seed=1).astype(np.float32 if c["dtype"] == "f32" else np.float64)
    d = Direct(c, x0, device=dev)
    clk = Clocks(local)
    clk.start()
    time.sleep(0.3)
    d.run(args.warmup)
    d.sync()
    K = args.steps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(d.stream)
    d.run(K)
    e1.record(d.stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    d.sync()
    inter = float(n) * (n - 1) * K / (ms / 1e3)
    peak = direct_peak(c)
    line = {"metric": "pair interactions/s (direct O(N^2) step, row f1)", "value": inter,
            "unit": "interactions/s", "n_gpus": 1, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": c["dtype"], "data": "synthetic (seeded normal X0)",
            "config": {"workload": f"{args.workload} model, direct step", "n": n, "d": c["d"],
                       "kernel": c["kernel"], "l2": "state fits in L2; no flush"},
            "particle_steps_per_s": n * K / (ms / 1e3),
            "roofline": {"bound": "alu", "kernel": "direct_kernel", "achieved": inter, "peak": peak,
                         "unit": "interactions/s", "frac": inter / peak, "traffic": None,
                         "peak_source": "derived: 148 SMs x 1.965 GHz x FMA-pipe lanes / pipe instructions per interaction"},
            "clocks": clocks, "gpu_launches": K, "e2e": None, "cpu_baseline": None}
    print(json.dumps(line), flush=True)
    return 0


def bench_partition(args, cfg, world, rank, local, dev, barrier, max_over_ranks):
    """One global system of world x n particles split by key range over the
    ranks.  Default: the library runs the whole step (kernels and
    NCCL exchanges in rbm_run, CUDA-graph replayed; records stored into the
    peers' buffers over NVLink when every rank could map them).
    --exchange torch: the caller-exchange protocol over torch.distributed."""
    import torch

    from paper_1812_10575_b200 import partition as PT
    K = args.steps
    gcfg = dict(cfg, n=cfg["n"] * world, replica=0)
    if args.exchange == "torch":
        ps = PT.PartitionedRBM(gcfg, world, [rank], PT.DistExchange(), device=dev)
        exchange = "torch.distributed all-to-all (caller exchanges)"
        if world <= 8 and ps.enable_fused():
            exchange = "torch.distributed counts/halo, records stored into peer buffers by the kernels"
        stream, launches = ps.systems[0].stream, ps.systems[0].launches_per_step
    else:
        ps = PT.CommPartitionedRBM(gcfg, world, rank, device=dev, fused=(args.exchange == "fused"))
        exchange = ("library NCCL counts/halo, records stored into peer buffers by the kernels over NVLink"
                    if ps.fused else "library NCCL all-to-all of the records")
        stream, launches = ps.stream, ps.launches_per_step
    clk = Clocks(local)
    clk.start()
    time.sleep(0.3)
    ps.run(args.warmup)
    ps.run(8)  # untimed: captures the CUDA graph of 8 steps the timed run replays
    ps.sync()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ps.run(K)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    ms = max_over_ranks(e0.elapsed_time(e1))
    ps.sync()
    value = gcfg["n"] * K / (ms / 1e3)
    # NVLink bytes each rank sends per step: the records leaving it (R B each,
    # (G-1)/G of its particles on average) + counts + halo
    R = rec_bytes(cfg)
    nvl = cfg["n"] * (world - 1) / world * R / (ms / K / 1e3) / 1e9
    line = {"metric": "particle-steps/s", "value": value, "unit": "particle-steps/s",
            "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": ms / K,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": cfg["dtype"], "data": "synthetic (Philox init from seed, BASELINE.json config)",
            "config": dict(config_dict(args, cfg, world), n_total=gcfg["n"],
                           multi_gpu="partitioned single system (key-range split, halo; " + exchange + ")"),
            "nvlink": {"records_gbs_per_gpu": nvl, "record_bytes": R,
                       "peak_gbs_per_direction": 770.0, "frac": nvl / 770.0,
                       "note": "bytes leaving each GPU per step / step time; peak = measured peer copy per direction (B200_PROFILING.md)"},
            "roofline": None, "clocks": clocks,
            "gpu_launches": launches * K, "e2e": None, "cpu_baseline": None,
            "note": "per-kernel roofline and e2e are reported by the 1-GPU run"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ps.close()
    import torch.distributed as dist
    dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1812_10575_b200 import RBM

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = workload(args, rank)
    dev = torch.device("cuda", local)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    if args.direct:
        return bench_direct(args, cfg, dev, local)
    mode = args.mode or ("partition" if world > 1 else "single")
    K = args.steps
    if mode == "partition":
        return bench_partition(args, cfg, world, rank, local, dev, barrier, max_over_ranks)
    s = RBM(cfg, device=dev)
    stream = s.stream
    clk = Clocks(local)
    clk.start()
    time.sleep(0.3)
    # warm-up right before the timed region (no idle gap: clocks stay up); it
    s.run(args.warmup)
    if s.layout[0] > 0 and args.steps >= 8:
        s.run(8)  # untimed: captures the CUDA graph of 8 steps the timed run replays
    s.sync()
    # timed region: K steps through rbm_run (the user API, graph-replayed)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    s.run(K)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    # per-kernel split: the same K steps again with the library's CUDA events
    # around every kernel (rbm_timing_begin: eager launches on the same stream)
    s.timing_begin(K)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    s.run(K)
    f1.record(stream)
    torch.cuda.synchronize()
    eager_ms = f0.elapsed_time(f1)
    clocks = clk.stop()
    per_kernel, nrec = s.timing_end()
    s.sync()
    lay = s.layout
    launches = s.launches_per_step * K if lay[0] > 0 else (K + 4095) // 4096
    n_total = cfg["n"] * world
    value = n_total * K / (ms / 1e3)

    # roofline of the dominant kernel (largest share of the step)
    name = max(per_kernel, key=per_kernel.get)
    avg_ms = per_kernel[name] / max(nrec, 1)
    peak, peak_kind = peaks()
    nbytes = alg_bytes(name, cfg)
    dbytes = design_bytes(name, cfg, lay)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(f"{args.workload}:p{cfg['p']}:{cfg['scheme']}:{name}")
    except Exception:
        pass
    if nbytes > 0:
        ach = nbytes / (avg_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": name, "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "peak_source": peak_kind, "traffic": traffic,
                "algorithmic_bytes_per_launch": nbytes, "avg_launch_ms": avg_ms,
                "algorithmic": "2 d s bytes per particle-step (SURVEY 8(d)) x N particles per launch",
                "design_bytes_per_launch": dbytes,
                "design_frac": (dbytes / (avg_ms / 1e3) / 1e9) / peak if dbytes else None}
        if name in ("rbmr_emit", "rbmr_seq_sweep"):
            roof["access"] = "random 32-byte sectors (x_{j_s} of randomly drawn particles): far below the streaming peak by nature"

    else:  # resident multi-step kernel (N <= 2048): latency-bound, no byte roofline
        roof = {"bound": "latency", "kernel": name, "achieved": None, "peak": None, "unit": "GB/s",
                "frac": None, "traffic": traffic, "avg_launch_ms": avg_ms,
                "note": "one CTA keeps the system in shared memory for many steps: bounded by barrier latency, not by HBM or ALU throughput"}
    step_ms = ms / K
    shares = {k: round(v / max(nrec, 1), 4) for k, v in per_kernel.items()}
    R = rec_bytes(cfg)
    useful = value / world * 2 * cfg["d"] * elt(cfg) / 1e9

    # end-to-end through the public API with host buffers (pinned)
    e2e = None
    if not args.no_e2e:
        npdt = np.float32 if cfg["dtype"] == "f32" else np.float64
        tdt = torch.float32 if cfg["dtype"] == "f32" else torch.float64
        hin = torch.empty((cfg["n"], cfg["d"]), dtype=tdt, pin_memory=True)
        hout = torch.empty((cfg["n"], cfg["d"]), dtype=tdt, pin_memory=True)
        s.gather(host=False)  # warm
        xin = hin.numpy()
        xin[:] = np.resize(RI.user_x0(min(cfg["n"], 1 << 20), cfg["d"], seed=rank).astype(npdt),
                           (cfg["n"], cfg["d"]))
        ue = s
        from paper_1812_10575_b200 import rbm as RB
        # one untimed pass of the same job first (graph capture for the K-step
        # chunking and the first host-copy setup are one-time costs)
        ue.set_state(xin)
        ue.run(K)
        RB.rbm_gather(ue.ctx, 0, cfg["n"], hout.data_ptr(), RB.MEM_HOST)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ue.set_state(xin)                       # pinned host -> device (inside the timed region)
        ue.run(K)                               # graph-replayed steps
        RB.rbm_gather(ue.ctx, 0, cfg["n"], hout.data_ptr(), RB.MEM_HOST)  # device -> pinned host
        t = time.perf_counter() - t0
        barrier()
        t = max_over_ranks(t)
        e2e = {"value": n_total * K / t, "unit": "particle-steps/s",
               "h2d_bytes_per_step": cfg["n"] * cfg["d"] * elt(cfg) / K,
               "d2h_bytes_per_step": cfg["n"] * cfg["d"] * elt(cfg) / K,
               "job": f"upload X0 from pinned host, {K} steps (rbm_run), download X_K to pinned host"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg)

    line = {"metric": "particle-steps/s", "value": value, "unit": "particle-steps/s",
            "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": cfg["dtype"], "data": "synthetic (Philox init from seed, BASELINE.json config)",
            "config": config_dict(args, cfg, world),
            "hbm": {"useful_gbs_per_gpu": useful, "useful_frac": useful / peak, "record_bytes": R,
                    "note": "useful = particle-steps/s x 2 d s (state read+write once), whole step"},
            "timing": {"headline": "rbm_run graph replays, CUDA events on the library stream",
                       "graph_capture_steps": 8 if (s.layout[0] > 0 and args.steps >= 8) else 0,
                       "eager_ms_per_step": eager_ms / K,
                       "per_kernel": "second window of K eager steps with library events around each kernel"},
            "layout": {"prefix_bits": s.layout[0], "passes": s.layout[1], "bucket_cap": s.layout[2]},
            "roofline": roof, "kernel_ms_per_step": shares, "clocks": clocks,
            "gpu_launches": launches, "e2e": e2e, "cpu_baseline": cpu}
    if rank == 0:
        print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
