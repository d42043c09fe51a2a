"""ctypes shim over oracle/liborbm_oracle.so -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  The product path
(paper_1812_10575_b200/) never does, and this module imports nothing from it.

The C source (oracle/rbm_oracle.c) is the oracle; this file only marshals
numpy arrays.  Configs are plain dicts with the keys of ``ORACLE_FIELDS``
(the same keys the product binding accepts, see rbm_inputs.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "rbm_oracle.c")
LIB = os.path.join(HERE, "librbm_oracle.so")

KERNELS = {"zero": 0, "dyson": 1, "coulomb": 2, "bounded_confidence": 3,
           "gauss_attr_rep": 4, "coulomb_reg": 5, "smooth": 6, "linear": 7, "adjacency": 8}
INITS = {"user": 0, "normal": 1, "box": 2, "sphere": 3, "mixture": 4, "abs_normal": 5}


class OracleCfg(C.Structure):
    _fields_ = [
        ("d", C.c_uint32), ("p", C.c_uint32), ("n", C.c_uint64),
        ("scheme", C.c_int32), ("integrator", C.c_int32), ("kernel", C.c_int32),
        ("potential", C.c_int32), ("constraint", C.c_int32), ("fp32", C.c_int32),
        ("init_kind", C.c_int32), ("replica", C.c_uint32), ("noise", C.c_int32),
        ("state_form", C.c_int32), ("pad1", C.c_int32),
        ("kparam", C.c_double * 4), ("vparam", C.c_double * 2), ("iparam", C.c_double * 8),
        ("sigma", C.c_double), ("dt", C.c_double), ("seed", C.c_uint64),
        ("adj_rp", C.c_void_p), ("adj_ci", C.c_void_p), ("adj_v", C.c_void_p), ("adj_nnz", C.c_uint64),
    ]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no fast-math: IEEE double)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared",
                               "-ffp-contract=off", "-o", LIB, SRC, "-lm"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        P = C.POINTER
        u32p, f64p, u64p = P(C.c_uint32), P(C.c_double), P(C.c_uint64)
        cfgp = P(OracleCfg)
        sig = {
            "oracle_philox4x32_10": (None, [u32p, u32p, u32p]),
            "oracle_u01_f32": (C.c_float, [C.c_uint32]),
            "oracle_u01_f64": (C.c_double, [C.c_uint32, C.c_uint32]),
            "oracle_noise": (None, [cfgp, C.c_uint32, C.c_uint64, f64p]),
            "oracle_kernel_eval": (None, [cfgp, f64p, f64p]),
            "oracle_init": (C.c_int, [cfgp, f64p]),
            "oracle_key": (C.c_uint32, [cfgp, C.c_uint32, C.c_uint64]),
            "oracle_permutation": (C.c_int, [cfgp, C.c_uint64, u32p]),
            "oracle_keys": (None, [cfgp, C.c_uint64, u32p]),
            "oracle_batches": (C.c_uint64, [C.c_uint64, C.c_uint32, u64p]),
            "oracle_batch_forces": (C.c_int, [cfgp, f64p, u32p, u64p, C.c_uint64, f64p]),
            "oracle_pair_flow": (None, [cfgp, f64p, f64p, C.c_double, f64p, f64p]),
            "oracle_rbm1_step": (C.c_int, [cfgp, C.c_uint64, f64p]),
            "oracle_batch_update": (C.c_int, [cfgp, C.c_uint64, u32p, f64p, C.c_uint32, f64p]),
            "oracle_direct_step": (C.c_int, [cfgp, C.c_uint64, f64p]),
            "oracle_slot_draw": (C.c_uint32, [cfgp, C.c_uint64, C.c_uint32, C.c_uint64]),
            "oracle_rbmr_slots": (C.c_int, [cfgp, C.c_uint64, u32p]),
            "oracle_rbmr_step": (C.c_int, [cfgp, C.c_uint64, f64p]),
            "oracle_rbmr_seq_step": (C.c_int, [cfgp, C.c_uint64, f64p]),
            "oracle_run": (C.c_int, [cfgp, C.c_uint64, C.c_uint64, f64p]),
            "oracle_direct_run": (C.c_int, [cfgp, C.c_uint64, C.c_uint64, f64p]),
            "oracle_adj_value": (C.c_double, [cfgp, C.c_uint32, C.c_uint32]),
            "oracle_adj_pair_flow": (None, [cfgp, C.c_uint32, C.c_uint32, f64p, f64p, C.c_double, f64p, f64p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def make_cfg(cfg: dict) -> OracleCfg:
    c = OracleCfg()
    c.d = int(cfg["d"])
    c.p = int(cfg["p"])
    c.n = int(cfg["n"])
    c.scheme = {"rbm1": 0, "rbmr": 1, "rbmr_seq": 2}[cfg.get("scheme", "rbm1")]
    c.integrator = {"em": 0, "split": 1, "verlet": 2}[cfg.get("integrator", "em")]
    c.state_form = {"xv": 0, "xx": 1}[cfg.get("state_form", "xv")]
    c.kernel = KERNELS[cfg["kernel"]]
    c.potential = {"none": 0, "harmonic": 1}[cfg.get("potential", "none")]
    c.constraint = {"none": 0, "sphere": 1}[cfg.get("constraint", "none")]
    c.fp32 = 1 if cfg.get("dtype", "f64") == "f32" else 0
    c.init_kind = INITS[cfg.get("init", "normal")]
    c.replica = int(cfg.get("replica", 0))
    c.noise = {"additive": 0, "geometric": 1}[cfg.get("noise", "additive")]
    for i, v in enumerate(cfg.get("kparam", [])):
        c.kparam[i] = float(v)
    vp = cfg.get("vparam", [1.0])
    for i, v in enumerate(vp):
        c.vparam[i] = float(v)
    for i, v in enumerate(cfg.get("iparam", [])):
        c.iparam[i] = float(v)
    c.sigma = float(cfg.get("sigma", 0.0))
    c.dt = float(cfg["dt"])
    c.seed = int(cfg.get("seed", 0)) & 0xFFFFFFFFFFFFFFFF
    adj = cfg.get("adjacency")
    if adj is not None:  # (row_ptr u32, col u32, val f64) numpy arrays, kept alive by the dict
        rp, ci, v = (np.ascontiguousarray(adj[0], dtype=np.uint32), np.ascontiguousarray(adj[1], dtype=np.uint32),
                     np.ascontiguousarray(adj[2], dtype=np.float64))
        cfg["_adj_keep"] = (rp, ci, v)
        c.adj_rp, c.adj_ci, c.adj_v = rp.ctypes.data, ci.ctypes.data, v.ctypes.data
        c.adj_nnz = len(ci)
    return c


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def philox(ctr, key):
    ctr = np.asarray(ctr, dtype=np.uint32)
    key = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(ctr, C.c_uint32), _p(key, C.c_uint32), _p(out, C.c_uint32))
    return out


def u01_f32(w: int) -> float:
    return float(lib().oracle_u01_f32(int(w)))


def u01_f64(a: int, b: int) -> float:
    return float(lib().oracle_u01_f64(int(a), int(b)))


def init(cfg: dict) -> np.ndarray:
    c = make_cfg(cfg)
    x = np.zeros((c.n, c.d), dtype=np.float64)
    rc = lib().oracle_init(C.byref(c), _p(x, C.c_double))
    if rc:
        raise ValueError(f"oracle_init rc={rc}")
    return x


def key(cfg: dict, i: int, m: int) -> int:
    return int(lib().oracle_key(C.byref(make_cfg(cfg)), int(i), int(m)))


def permutation(cfg: dict, m: int) -> np.ndarray:
    c = make_cfg(cfg)
    order = np.zeros(c.n, dtype=np.uint32)
    lib().oracle_permutation(C.byref(c), int(m), _p(order, C.c_uint32))
    return order


def keys(cfg: dict, m: int) -> np.ndarray:
    c = make_cfg(cfg)
    out = np.zeros(c.n, dtype=np.uint32)
    lib().oracle_keys(C.byref(c), int(m), _p(out, C.c_uint32))
    return out


def batch_starts(n: int, p: int) -> np.ndarray:
    nb = lib().oracle_batches(int(n), int(p), None)
    s = np.zeros(nb + 1, dtype=np.uint64)
    lib().oracle_batches(int(n), int(p), _p(s, C.c_uint64))
    return s


def batch_forces(cfg: dict, x: np.ndarray, order: np.ndarray, starts=None) -> np.ndarray:
    c = make_cfg(cfg)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(c.n, c.d)
    order = np.ascontiguousarray(order, dtype=np.uint32)
    if starts is None:
        starts = batch_starts(c.n, c.p)
    starts = np.ascontiguousarray(starts, dtype=np.uint64)
    f = np.zeros_like(x)
    lib().oracle_batch_forces(C.byref(c), _p(x, C.c_double), _p(order, C.c_uint32),
                              _p(starts, C.c_uint64), len(starts) - 1, _p(f, C.c_double))
    return f


def kernel_eval(cfg: dict, z) -> np.ndarray:
    c = make_cfg(cfg)
    z = np.ascontiguousarray(z, dtype=np.float64).reshape(c.d)
    out = np.zeros(c.d)
    lib().oracle_kernel_eval(C.byref(c), _p(z, C.c_double), _p(out, C.c_double))
    return out


def noise(cfg: dict, i: int, m: int) -> np.ndarray:
    c = make_cfg(cfg)
    z = np.zeros(c.d)
    lib().oracle_noise(C.byref(c), int(i), int(m), _p(z, C.c_double))
    return z


def pair_flow(cfg: dict, xi, xj, tau: float):
    c = make_cfg(cfg)
    xi = np.ascontiguousarray(xi, dtype=np.float64).reshape(c.d)
    xj = np.ascontiguousarray(xj, dtype=np.float64).reshape(c.d)
    yi, yj = np.zeros(c.d), np.zeros(c.d)
    lib().oracle_pair_flow(C.byref(c), _p(xi, C.c_double), _p(xj, C.c_double), float(tau),
                           _p(yi, C.c_double), _p(yj, C.c_double))
    return yi, yj


def _stepper(name):
    def f(cfg: dict, x: np.ndarray, m: int) -> np.ndarray:
        c = make_cfg(cfg)
        y = np.array(x, dtype=np.float64, copy=True).reshape(c.n, c.d)
        rc = getattr(lib(), name)(C.byref(c), int(m), _p(y, C.c_double))
        if rc:
            raise ValueError(f"{name} rc={rc}")
        return y
    return f


rbm1_step = _stepper("oracle_rbm1_step")
direct_step = _stepper("oracle_direct_step")
rbmr_step = _stepper("oracle_rbmr_step")
rbmr_seq_step = _stepper("oracle_rbmr_seq_step")


def run(cfg: dict, x: np.ndarray, m0: int, nsteps: int) -> np.ndarray:
    c = make_cfg(cfg)
    y = np.array(x, dtype=np.float64, copy=True).reshape(c.n, c.d)
    rc = lib().oracle_run(C.byref(c), int(m0), int(nsteps), _p(y, C.c_double))
    if rc:
        raise ValueError(f"oracle_run rc={rc}")
    return y


def direct_run(cfg: dict, x: np.ndarray, m0: int, nsteps: int) -> np.ndarray:
    c = make_cfg(cfg)
    y = np.array(x, dtype=np.float64, copy=True).reshape(c.n, c.d)
    rc = lib().oracle_direct_run(C.byref(c), int(m0), int(nsteps), _p(y, C.c_double))
    if rc:
        raise ValueError(f"oracle_direct_run rc={rc}")
    return y


def slot_draw(cfg: dict, s: int, t: int, m: int) -> int:
    return int(lib().oracle_slot_draw(C.byref(make_cfg(cfg)), int(s), int(t), int(m)))


def rbmr_slots(cfg: dict, m: int) -> np.ndarray:
    c = make_cfg(cfg)
    nb = (c.n + c.p - 1) // c.p
    js = np.zeros(nb * c.p, dtype=np.uint32)
    lib().oracle_rbmr_slots(C.byref(c), int(m), _p(js, C.c_uint32))
    return js


def adj_value(cfg: dict, i: int, j: int) -> float:
    return float(lib().oracle_adj_value(C.byref(make_cfg(cfg)), int(i), int(j)))


def adj_pair_flow(cfg: dict, i: int, j: int, xi, xj, tau: float):
    c = make_cfg(cfg)
    xi = np.ascontiguousarray(xi, dtype=np.float64).reshape(c.d)
    xj = np.ascontiguousarray(xj, dtype=np.float64).reshape(c.d)
    yi, yj = np.zeros(c.d), np.zeros(c.d)
    lib().oracle_adj_pair_flow(C.byref(c), int(i), int(j), _p(xi, C.c_double), _p(xj, C.c_double), float(tau),
                               _p(yi, C.c_double), _p(yj, C.c_double))
    return yi, yj


def batch_update(cfg: dict, m: int, ids, xb) -> np.ndarray:
    """One batch of Alg. 1 (members in sorted order) -> their X_{m+1}."""
    c = make_cfg(cfg)
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    xb = np.ascontiguousarray(xb, dtype=np.float64).reshape(len(ids), c.d)
    xo = np.zeros_like(xb)
    rc = lib().oracle_batch_update(C.byref(c), int(m), _p(ids, C.c_uint32), _p(xb, C.c_double),
                                   len(ids), _p(xo, C.c_double))
    if rc:
        raise ValueError(f"oracle_batch_update rc={rc}")
    return xo
