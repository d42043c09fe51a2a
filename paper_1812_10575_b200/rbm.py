"""Thin ctypes binding of librbm.so (include/rbm.h) -- argument marshalling only.

Every step of the RBM path runs in the library's CUDA kernels.  PyTorch is
used for device memory (the caller-owned workspace and output tensors) and
for the CUDA stream handle.  There is no CPU fallback: if librbm.so is
missing or cannot be loaded, importing a symbol raises.

Low-level names mirror the C ABI (rbm_init, rbm_step, ...); ``RBM`` is a
small convenience wrapper that allocates the workspace with torch.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# RBM_LIB: an alternative in-tree build of the same library (design experiments)
LIB_PATH = os.environ.get("RBM_LIB") or os.path.join(PKG, "librbm.so")

RBM_ABI_VERSION = 1
STATUS = {0: "RBM_OK", 1: "RBM_ERR_INVALID_ARG", 2: "RBM_ERR_UNKNOWN_KERNEL",
          3: "RBM_ERR_UNSUPPORTED", 4: "RBM_ERR_WORKSPACE", 5: "RBM_ERR_CUDA",
          6: "RBM_ERR_NCCL", 7: "RBM_ERR_NONFINITE", 8: "RBM_ERR_STATE", 9: "RBM_ERR_CAPACITY"}
KERNELS = {"zero": 0, "dyson": 1, "coulomb": 2, "bounded_confidence": 3,
           "gauss_attr_rep": 4, "coulomb_reg": 5, "smooth": 6, "linear": 7, "adjacency": 8}
INITS = {"user": 0, "normal": 1, "box": 2, "sphere": 3, "mixture": 4, "abs_normal": 5}
NOISES = {"additive": 0, "geometric": 1}
MEM_DEVICE, MEM_HOST = 0, 1
EXPORTS = ["rbm_workspace_size", "rbm_init", "rbm_set_state", "rbm_step", "rbm_run",
           "rbm_gather", "rbm_sync", "rbm_step_index", "rbm_launches_per_step", "rbm_layout",
           "rbm_debug_permutation", "rbm_debug_slots", "rbm_debug_philox", "rbm_last_error",
           "rbm_destroy", "rbm_kernel_name", "rbm_timing_begin", "rbm_timing_end",
           "rbm_part_info_get", "rbm_part_prologue", "rbm_part_phase1", "rbm_part_phase2",
           "rbm_part_set_peers", "rbm_part_map_peers", "rbm_get_nccl_unique_id", "rbm_gather_local",
           "rbm_part_phase", "rbm_set_adjacency",
           "rbm_direct_workspace_size", "rbm_direct_reset", "rbm_direct_run", "rbm_direct_sync"]


class RbmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class RbmConfig(C.Structure):
    _fields_ = [
        ("abi_version", C.c_uint32), ("dtype", C.c_uint32), ("d", C.c_uint32), ("p", C.c_uint32),
        ("n", C.c_uint64),
        ("scheme", C.c_uint32), ("integrator", C.c_uint32), ("kernel", C.c_uint32),
        ("potential", C.c_uint32), ("constraint", C.c_uint32), ("init", C.c_uint32),
        ("kparam", C.c_double * 4), ("vparam", C.c_double * 2), ("iparam", C.c_double * 8),
        ("sigma", C.c_double), ("dt", C.c_double), ("seed", C.c_uint64), ("step0", C.c_uint64),
        ("replica", C.c_uint32), ("world_size", C.c_int32), ("rank", C.c_int32),
        ("debug_bucket_cap", C.c_uint32), ("noise", C.c_uint32), ("state_form", C.c_uint32),
    ]


_lib = None


def lib():
    """Load librbm.so (fails loudly if it is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built; run `python -m paper_1812_10575_b200.build`")
        L = C.CDLL(LIB_PATH)
        vp, cfgp, u32, u64, st = C.c_void_p, C.POINTER(RbmConfig), C.c_uint32, C.c_uint64, C.c_int
        sig = {
            "rbm_workspace_size": (st, [cfgp, C.POINTER(C.c_size_t)]),
            "rbm_init": (st, [cfgp, vp, C.c_size_t, vp, vp, C.POINTER(vp)]),
            "rbm_set_state": (st, [vp, vp, u32]),
            "rbm_step": (st, [vp]),
            "rbm_run": (st, [vp, u64]),
            "rbm_gather": (st, [vp, u64, u64, vp, u32]),
            "rbm_sync": (st, [vp]),
            "rbm_step_index": (u64, [vp]),
            "rbm_launches_per_step": (u32, [vp]),
            "rbm_layout": (st, [vp, C.POINTER(u32), C.POINTER(u32), C.POINTER(u32)]),
            "rbm_debug_permutation": (st, [vp, vp]),
            "rbm_debug_slots": (st, [vp, vp]),
            "rbm_debug_philox": (st, [vp, vp, u64, vp]),
            "rbm_last_error": (C.c_char_p, [vp]),
            "rbm_destroy": (st, [vp]),
            "rbm_kernel_name": (C.c_char_p, [vp, u32]),
            "rbm_timing_begin": (st, [vp, u32]),
            "rbm_timing_end": (st, [vp, C.POINTER(C.c_double), C.POINTER(u32)]),
            "rbm_get_nccl_unique_id": (st, [vp]),
            "rbm_gather_local": (st, [vp, vp, vp, C.POINTER(u64)]),
            "rbm_part_map_peers": (st, [vp]),
            "rbm_set_adjacency": (st, [vp, vp, vp, vp, u64]),
            "rbm_direct_workspace_size": (st, [cfgp, C.POINTER(C.c_size_t)]),
            "rbm_direct_reset": (st, [cfgp, vp, vp]),
            "rbm_direct_run": (st, [cfgp, vp, u64, u64, vp, C.c_size_t, vp]),
            "rbm_direct_sync": (st, [cfgp, vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def _check(status: int, ctx=None):
    if status != 0:
        msg = lib().rbm_last_error(ctx)
        raise RbmError(status, msg.decode() if msg else "")


def make_config(cfg: dict) -> RbmConfig:
    """Build the C struct from a workload dict (rbm_inputs.py keys)."""
    c = RbmConfig()
    c.abi_version = RBM_ABI_VERSION
    c.dtype = {"f32": 0, "f64": 1}[cfg.get("dtype", "f64")]
    c.d = int(cfg["d"])
    c.p = int(cfg["p"])
    c.n = int(cfg["n"])
    c.scheme = {"rbm1": 0, "rbmr": 1, "rbmr_seq": 2}[cfg.get("scheme", "rbm1")]
    c.integrator = {"em": 0, "split": 1, "verlet": 2}[cfg.get("integrator", "em")]
    c.state_form = {"xv": 0, "xx": 1}[cfg.get("state_form", "xv")]
    c.kernel = KERNELS[cfg["kernel"]] if isinstance(cfg["kernel"], str) else int(cfg["kernel"])
    c.potential = {"none": 0, "harmonic": 1}[cfg.get("potential", "none")]
    c.constraint = {"none": 0, "sphere": 1}[cfg.get("constraint", "none")]
    c.init = INITS[cfg.get("init", "normal")]
    for i, v in enumerate(cfg.get("kparam", [])):
        c.kparam[i] = float(v)
    for i, v in enumerate(cfg.get("vparam", [1.0])):
        c.vparam[i] = float(v)
    for i, v in enumerate(cfg.get("iparam", [])):
        c.iparam[i] = float(v)
    c.sigma = float(cfg.get("sigma", 0.0))
    c.dt = float(cfg["dt"])
    c.seed = int(cfg.get("seed", 0)) & 0xFFFFFFFFFFFFFFFF
    c.step0 = int(cfg.get("step0", 0))
    c.replica = int(cfg.get("replica", 0))
    c.world_size = int(cfg.get("world_size", 1))
    c.rank = int(cfg.get("rank", 0))
    c.debug_bucket_cap = int(cfg.get("debug_bucket_cap", 0))
    c.noise = NOISES[cfg.get("noise", "additive")]
    return c


# ---------------------------------------------------------------- C names
def rbm_workspace_size(cfg: RbmConfig) -> int:
    n = C.c_size_t(0)
    _check(lib().rbm_workspace_size(C.byref(cfg), C.byref(n)))
    return n.value


def rbm_get_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().rbm_get_nccl_unique_id(buf))
    return buf.raw


def rbm_init(cfg: RbmConfig, ws_ptr: int, ws_bytes: int, stream: int = 0, nccl_id: bytes | None = None):
    out = C.c_void_p()
    idbuf = C.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
    _check(lib().rbm_init(C.byref(cfg), C.c_void_p(ws_ptr), ws_bytes, C.c_void_p(stream), idbuf,
                          C.byref(out)))
    return out


def rbm_gather_local(ctx, ids_ptr: int, x_ptr: int) -> int:
    n = C.c_uint64(0)
    _check(lib().rbm_gather_local(ctx, C.c_void_p(ids_ptr), C.c_void_p(x_ptr), C.byref(n)), ctx)
    return n.value


def rbm_part_map_peers(ctx):
    _check(lib().rbm_part_map_peers(ctx), ctx)


def rbm_set_state(ctx, x_ptr: int, where: int):
    _check(lib().rbm_set_state(ctx, C.c_void_p(x_ptr), where), ctx)


def rbm_step(ctx):
    _check(lib().rbm_step(ctx), ctx)


def rbm_run(ctx, nsteps: int):
    _check(lib().rbm_run(ctx, int(nsteps)), ctx)


def rbm_gather(ctx, id_begin: int, id_end: int, x_ptr: int, where: int):
    _check(lib().rbm_gather(ctx, int(id_begin), int(id_end), C.c_void_p(x_ptr), where), ctx)


def rbm_sync(ctx):
    _check(lib().rbm_sync(ctx), ctx)


def rbm_step_index(ctx) -> int:
    return int(lib().rbm_step_index(ctx))


def rbm_launches_per_step(ctx) -> int:
    return int(lib().rbm_launches_per_step(ctx))


def rbm_layout(ctx):
    a, b, c = C.c_uint32(), C.c_uint32(), C.c_uint32()
    _check(lib().rbm_layout(ctx, C.byref(a), C.byref(b), C.byref(c)), ctx)
    return a.value, b.value, c.value


def rbm_debug_permutation(ctx, out_ptr: int):
    _check(lib().rbm_debug_permutation(ctx, C.c_void_p(out_ptr)), ctx)


def rbm_debug_slots(ctx, out_ptr: int):
    _check(lib().rbm_debug_slots(ctx, C.c_void_p(out_ptr)), ctx)


def rbm_debug_philox(in_ptr: int, out_ptr: int, count: int, stream: int = 0):
    _check(lib().rbm_debug_philox(C.c_void_p(in_ptr), C.c_void_p(out_ptr), int(count),
                                  C.c_void_p(stream)))


def rbm_kernel_name(ctx, i: int) -> str:
    return lib().rbm_kernel_name(ctx, int(i)).decode()


def rbm_timing_begin(ctx, max_steps: int):
    _check(lib().rbm_timing_begin(ctx, int(max_steps)), ctx)


def rbm_timing_end(ctx):
    """-> (dict kernel name -> summed ms, steps recorded)"""
    k = rbm_launches_per_step(ctx)
    arr = (C.c_double * max(k, 1))()
    steps = C.c_uint32()
    _check(lib().rbm_timing_end(ctx, arr, C.byref(steps)), ctx)
    return {rbm_kernel_name(ctx, i): arr[i] for i in range(k)}, steps.value


def rbm_destroy(ctx):
    _check(lib().rbm_destroy(ctx))


# ----------------------------------------------------------- convenience
class RBM:
    """One RBM system on the current CUDA device (torch provides memory/stream)."""

    def __init__(self, cfg: dict, x0=None, device=None, nccl_id: bytes | None = None):
        import torch
        self.torch = torch
        self.cfg = dict(cfg)
        if x0 is not None:
            self.cfg["init"] = "user"
        self.c = make_config(self.cfg)
        self.device = torch.device(device or "cuda")
        self.dtype = torch.float64 if self.cfg.get("dtype", "f64") == "f64" else torch.float32
        self.n, self.d = int(self.c.n), int(self.c.d)
        # rows this context takes in set_state: its initial id range (all N on one GPU)
        G, r = int(self.c.world_size), int(self.c.rank)
        self.id0 = self.n * r // G
        self.n_rows = self.n * (r + 1) // G - self.id0
        self.ws_bytes = rbm_workspace_size(self.c)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        self.stream = torch.cuda.current_stream(self.device)
        self.ctx = rbm_init(self.c, self.ws.data_ptr(), self.ws_bytes, self.stream.cuda_stream, nccl_id)
        adj = self.cfg.get("adjacency")
        if adj is not None:  # clustering model: CSR adjacency uploaded once, kept by this object
            rp, ci, v = adj[0], adj[1], adj[2]
            self._adj = (torch.as_tensor(rp.astype("int64")).to(torch.int32).to(self.device),
                         torch.as_tensor(ci.astype("int64")).to(torch.int32).to(self.device),
                         torch.as_tensor(v, dtype=torch.float64).to(self.device))
            _check(lib().rbm_set_adjacency(self.ctx, C.c_void_p(self._adj[0].data_ptr()),
                                           C.c_void_p(self._adj[1].data_ptr()),
                                           C.c_void_p(self._adj[2].data_ptr()), len(ci)), self.ctx)
        if x0 is not None:
            self.set_state(x0)

    def set_state(self, x):
        torch = self.torch
        if isinstance(x, torch.Tensor) and x.is_cuda:
            t = x.to(self.dtype).contiguous()
            rbm_set_state(self.ctx, t.data_ptr(), MEM_DEVICE)
            self._keep = t
        else:
            import numpy as np
            a = np.ascontiguousarray(np.asarray(x), dtype=np.float64 if self.dtype == torch.float64 else np.float32)
            assert a.size == self.n_rows * self.d
            rbm_set_state(self.ctx, a.ctypes.data, MEM_HOST)

    def step(self):
        rbm_step(self.ctx)

    def run(self, nsteps: int):
        rbm_run(self.ctx, nsteps)

    def sync(self):
        rbm_sync(self.ctx)

    def gather(self, id_begin: int = 0, id_end: int | None = None, host: bool = False):
        torch = self.torch
        id_end = self.n if id_end is None else id_end
        if host:
            import numpy as np
            out = np.empty((id_end - id_begin, self.d),
                           dtype=np.float64 if self.dtype == torch.float64 else np.float32)
            rbm_gather(self.ctx, id_begin, id_end, out.ctypes.data, MEM_HOST)
            return out
        out = torch.empty((id_end - id_begin, self.d), dtype=self.dtype, device=self.device)
        rbm_gather(self.ctx, id_begin, id_end, out.data_ptr(), MEM_DEVICE)
        return out

    def gather_local(self):
        """(ids, x): the particles this context holds, unordered (device tensors)."""
        torch = self.torch
        cap = self.n  # a rank never holds more than the global N
        ids = torch.empty(cap, dtype=torch.int32, device=self.device)
        x = torch.empty((cap, self.d), dtype=self.dtype, device=self.device)
        k = rbm_gather_local(self.ctx, ids.data_ptr(), x.data_ptr())
        return ids[:k], x[:k]

    def step_permutation(self):
        """One rbm_step that also returns its permutation (sorted position -> id)."""
        out = self.torch.full((self.n,), -1, dtype=self.torch.int32, device=self.device)
        rbm_debug_permutation(self.ctx, out.data_ptr())
        rbm_step(self.ctx)
        self.stream.synchronize()
        return out.cpu().numpy().view("uint32")

    def slots(self):
        """Slot draws j_s of the last step (partitioned: this rank's batches)."""
        nb = (self.n + self.c.p - 1) // self.c.p
        G, r = int(self.c.world_size), int(self.c.rank)
        nown = (nb * (r + 1) // G - nb * r // G) * self.c.p
        out = self.torch.empty(nown, dtype=self.torch.int32, device=self.device)
        rbm_debug_slots(self.ctx, out.data_ptr())
        self.stream.synchronize()
        return out.cpu().numpy().view("uint32")

    def timing_begin(self, max_steps: int):
        rbm_timing_begin(self.ctx, max_steps)

    def timing_end(self):
        return rbm_timing_end(self.ctx)

    @property
    def step_index(self) -> int:
        return rbm_step_index(self.ctx)

    @property
    def launches_per_step(self) -> int:
        return rbm_launches_per_step(self.ctx)

    @property
    def layout(self):
        return rbm_layout(self.ctx)

    def close(self):
        if getattr(self, "ctx", None):
            rbm_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------ direct O(N^2) steps (f1)
class Direct:
    """Fully coupled Euler-Maruyama steps (rbm_direct_run) on an id-ordered
    device tensor (N x d), synchronously coupled with RBM runs of the same seed."""

    def __init__(self, cfg: dict, x, device=None):
        import torch
        self.torch = torch
        self.c = make_config(dict(cfg, p=2, scheme="rbm1", world_size=1, rank=0))
        self.c.n = int(cfg["n"])
        self.device = torch.device(device or "cuda")
        self.dtype = torch.float64 if cfg.get("dtype", "f64") == "f64" else torch.float32
        n = C.c_size_t(0)
        _check(lib().rbm_direct_workspace_size(C.byref(self.c), C.byref(n)))
        self.ws_bytes = n.value
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        self.stream = torch.cuda.current_stream(self.device)
        self.x = torch.as_tensor(x, dtype=self.dtype).to(self.device).contiguous().reshape(self.c.n, self.c.d)
        _check(lib().rbm_direct_reset(C.byref(self.c), C.c_void_p(self.ws.data_ptr()),
                                      C.c_void_p(self.stream.cuda_stream)))
        self.step_index = int(cfg.get("step0", 0))

    def run(self, nsteps: int):
        _check(lib().rbm_direct_run(C.byref(self.c), C.c_void_p(self.x.data_ptr()), self.step_index,
                                    int(nsteps), C.c_void_p(self.ws.data_ptr()), self.ws_bytes,
                                    C.c_void_p(self.stream.cuda_stream)))
        self.step_index += int(nsteps)

    def sync(self):
        _check(lib().rbm_direct_sync(C.byref(self.c), C.c_void_p(self.ws.data_ptr()),
                                     C.c_void_p(self.stream.cuda_stream)))

    def gather(self):
        self.sync()
        return self.x.cpu().numpy()
