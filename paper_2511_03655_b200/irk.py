"""Thin Python binding of the C ABI in include/irk.h (argument marshalling only).

Every step of the integration runs in paper_2511_03655_b200/lib/libirk.so;
PyTorch only provides device memory and streams.  There is no CPU fallback:
if the library is missing this module raises on import of the library.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

KEPLER, NBODY, FPU_BETA, HENON_HEILES, NBODY_DIRECT, SCHWARZSCHILD = 1, 2, 3, 4, 5, 6
OK, W_MAXITER, E_ARG, E_CUDA, E_DIVERGED, E_COMM, E_STATE = 0, 1, -1, -2, -3, -4, -5
OPT_MODE, OPT_MAX_ITERS, OPT_ENERGY_EVERY, OPT_MAPPING, OPT_BALANCE, OPT_VSHARDS = 1, 2, 3, 4, 5, 6
OPT_LOCAL_ENERGY = 7
OPT_SCHEDULE = 8
MAP_AUTO, MAP_G1, MAP_G2, MAP_G4, MAP_G8, MAP_G8M = 0, 1, 2, 4, 8, 9  # IRK_OPT_MAPPING (include/irk.h)
OPT_DEVICE_LOOP = 9
OPT_EXCHANGE = 10  # IRK_NBODY_DIRECT under set_comm: 0 = ncclAllGather, 1 = fused NVLink stores
EXCHANGE_ALLGATHER, EXCHANGE_FUSED = 0, 1
INFO_DEVICE_LOOP_USED = 100
INFO_MAPPING_USED = 101
PARTITIONED, FIRST_ORDER = 0, 1

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IRK_LIB_OVERRIDE") or os.path.join(_HERE, "lib", "libirk.so")  # override: A/B builds only

SYMBOLS = ["irk_create", "irk_set_params", "irk_set_option", "irk_workspace_bytes",
           "irk_integrate", "irk_integrate_host", "irk_energy", "irk_stats", "irk_tableau",
           "irk_set_comm", "irk_nccl_unique_id", "irk_last_error", "irk_destroy", "irk_probe_dfma",
           "irk_probe_divsqrt", "irk_local_energy_error", "irk_get_option"]

_lib = None
_lock = threading.Lock()


class IrkError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"irk error {code}: {msg}")
        self.code = code


def lib():
    """Load libirk.so (raises if it was not built: no fallback path exists)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} missing: run paper_2511_03655_b200/build.py "
                                  "(the CUDA library is the only implementation)")
            l = ctypes.CDLL(LIB_PATH)
            vp, dp, i64p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
            l.irk_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int64, ctypes.c_int64]
            l.irk_create.restype = vp
            l.irk_set_params.argtypes = [vp, dp, ctypes.c_int]
            l.irk_set_option.argtypes = [vp, ctypes.c_int, ctypes.c_int64]
            l.irk_workspace_bytes.argtypes = [vp]
            l.irk_workspace_bytes.restype = ctypes.c_size_t
            l.irk_integrate.argtypes = [vp, vp, ctypes.c_double, vp, vp, vp, vp]
            l.irk_integrate_host.argtypes = [vp, dp, ctypes.c_double, dp, i64p, vp]
            l.irk_energy.argtypes = [vp, vp, vp, vp]
            l.irk_stats.argtypes = [vp, vp, vp, i64p]
            l.irk_tableau.argtypes = [dp, dp, dp, dp]
            l.irk_set_comm.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int]
            l.irk_nccl_unique_id.argtypes = [vp]
            l.irk_last_error.argtypes = [vp]
            l.irk_last_error.restype = ctypes.c_char_p
            l.irk_destroy.argtypes = [vp]
            l.irk_probe_dfma.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp]
            l.irk_probe_dfma.restype = ctypes.c_int64
            l.irk_probe_divsqrt.argtypes = [vp, vp, vp, ctypes.c_int64, vp]
            l.irk_local_energy_error.argtypes = [vp, vp, vp, vp]
            l.irk_get_option.argtypes = [vp, ctypes.c_int, i64p]
            _lib = l
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def tableau():
    """The fp64 (c, b, mu, nu) the kernels use (library's own __float128 build)."""
    c, b, mu, nu = np.zeros(8), np.zeros(8), np.zeros((8, 8)), np.zeros((8, 8))
    rc = lib().irk_tableau(_dp(c), _dp(b), _dp(mu), _dp(nu))
    if rc:
        raise IrkError(rc, "irk_tableau")
    return c, b, mu, nu


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _need(t, name, dtype, shape=None, device=None, min_numel=None):
    """Explicit checks of a device buffer before its raw pointer crosses the C ABI
    (which cannot see sizes): dtype, CUDA, contiguity, shape / size, device.
    Raises ValueError (not assert: survives python -O)."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name}: expected a torch tensor, got {type(t).__name__}")
    if t.dtype != dtype:
        raise ValueError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if not t.is_cuda:
        raise ValueError(f"{name}: must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    if device is not None and t.device != device:
        raise ValueError(f"{name}: on {t.device}, expected {device}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    if min_numel is not None and t.numel() < min_numel:
        raise ValueError(f"{name}: {t.numel()} elements, need >= {min_numel}")


class Integrator:
    """One irk_ctx.  y tensors are float64 (dim, batch), contiguous, on CUDA."""

    def __init__(self, problem: int, dim: int, h: float, nsteps: int, batch: int, params,
                 *, mode: int | None = None, max_iters: int = 100, energy_every: int = 0,
                 mapping: int = 0, balance: int = -1, vshards: int = 1, local_energy: bool = False,
                 schedule: int = 0, device_loop: int = 1, exchange: int = 0):
        L = lib()
        self._ctx = L.irk_create(problem, dim, h, nsteps, batch)
        if not self._ctx:
            raise IrkError(E_ARG, L.irk_last_error(None).decode())
        self.problem, self.dim, self.h, self.nsteps, self.batch = problem, dim, h, nsteps, batch
        self.energy_every = energy_every
        p = np.ascontiguousarray(params, dtype=np.float64)
        self._check(L.irk_set_params(self._ctx, _dp(p), len(p)))
        if mode is not None:  # default: the library's (partitioned; first-order for SCHWARZSCHILD)
            self._check(L.irk_set_option(self._ctx, OPT_MODE, mode))
        for key, val in ((OPT_MAX_ITERS, max_iters),
                         (OPT_ENERGY_EVERY, energy_every), (OPT_MAPPING, mapping),
                         (OPT_BALANCE, balance), (OPT_SCHEDULE, schedule)):
            self._check(L.irk_set_option(self._ctx, key, val))
        if vshards != 1:
            self._check(L.irk_set_option(self._ctx, OPT_VSHARDS, vshards))
        if local_energy:
            self._check(L.irk_set_option(self._ctx, OPT_LOCAL_ENERGY, 1))
        if problem == NBODY_DIRECT:
            self._check(L.irk_set_option(self._ctx, OPT_DEVICE_LOOP, device_loop))
            self._check(L.irk_set_option(self._ctx, OPT_EXCHANGE, exchange))
        self.rank, self.nranks = 0, 1

    def set_comm(self, unique_id: bytes, rank: int, nranks: int):
        """Body-shard an IRK_NBODY_DIRECT system over NCCL (include/irk.h irk_set_comm)."""
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        self._check(lib().irk_set_comm(self._ctx, ctypes.cast(buf, ctypes.c_void_p), rank, nranks))
        self.rank, self.nranks = rank, nranks

    @property
    def local_dim(self) -> int:
        return self.dim // self.nranks

    def _check(self, rc):
        if rc < 0:
            raise IrkError(rc, lib().irk_last_error(self._ctx).decode())
        return rc

    def close(self):
        if getattr(self, "_ctx", None):
            lib().irk_destroy(self._ctx)
            self._ctx = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def workspace_bytes(self) -> int:
        return int(lib().irk_workspace_bytes(self._ctx))

    def new_workspace(self, device="cuda"):
        import torch
        return torch.zeros(self.workspace_bytes, dtype=torch.uint8, device=device)

    def n_energy(self) -> int:
        return self.nsteps // self.energy_every + 1 if self.energy_every > 0 else 0

    def integrate(self, y, workspace, *, t0: float = 0.0, energy=None, iters=None, stream=None):
        """Advance y in place on the device (irk_integrate); asynchronous on `stream`."""
        import torch
        _need(y, "y", torch.float64, shape=(self.local_dim, self.batch))
        _need(workspace, "workspace", torch.uint8, device=y.device, min_numel=self.workspace_bytes)
        if self.energy_every > 0 and energy is None:
            raise ValueError("energy: required when energy_every > 0")
        if self.energy_every <= 0:
            energy = None          # no samples are written
        if energy is not None:
            _need(energy, "energy", torch.float64, shape=(self.n_energy(), self.batch), device=y.device)
        if iters is not None:
            _need(iters, "iters", torch.int64, shape=(self.batch,), device=y.device)
        s = torch.cuda.current_stream(y.device) if stream is None else stream
        self._check(lib().irk_integrate(self._ctx, _ptr(y), t0, _ptr(workspace), _ptr(energy),
                                        _ptr(iters), ctypes.c_void_p(s.cuda_stream)))

    def integrate_host(self, y_host: np.ndarray, *, t0: float = 0.0, want_energy=True,
                       want_iters=True, stream=None):
        """End-to-end call from host memory (irk_integrate_host); returns (energy, iters)."""
        import torch
        if not (isinstance(y_host, np.ndarray) and y_host.dtype == np.float64 and y_host.flags.c_contiguous
                and y_host.shape == (self.local_dim, self.batch)):
            raise ValueError(f"y_host: need a C-contiguous float64 ndarray of shape {(self.local_dim, self.batch)}")
        E = np.zeros((self.n_energy(), self.batch)) if (want_energy and self.energy_every > 0) else None
        it = np.zeros(self.batch, dtype=np.int64) if want_iters else None
        s = torch.cuda.current_stream() if stream is None else stream
        self._check(lib().irk_integrate_host(
            self._ctx, _dp(y_host), t0, _dp(E) if E is not None else None,
            it.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)) if it is not None else None,
            ctypes.c_void_p(s.cuda_stream)))
        return E, it

    def energy(self, y, out=None, stream=None):
        import torch
        _need(y, "y", torch.float64, shape=(self.local_dim, self.batch))
        if out is None:
            out = torch.empty(self.batch, dtype=torch.float64, device=y.device)
        _need(out, "out", torch.float64, shape=(self.batch,), device=y.device)
        s = torch.cuda.current_stream(y.device) if stream is None else stream
        self._check(lib().irk_energy(self._ctx, _ptr(y), _ptr(out), ctypes.c_void_p(s.cuda_stream)))
        return out

    def stats(self, workspace, stream=None):
        import torch
        _need(workspace, "workspace", torch.uint8, min_numel=self.workspace_bytes)
        out = np.zeros(4, dtype=np.int64)
        s = torch.cuda.current_stream(workspace.device) if stream is None else stream
        rc = lib().irk_stats(self._ctx, _ptr(workspace), ctypes.c_void_p(s.cuda_stream),
                             out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
        if rc < 0 and rc != E_DIVERGED:  # E_DIVERGED is a device outcome, not a call error
            self._check(rc)
        return rc, dict(maxiter_traj=int(out[0]), diverged_traj=int(out[1]),
                        first_bad_step=int(out[2]), total_sweeps=int(out[3]))

    def set_option(self, key: int, val: int):
        """irk_set_option (include/irk.h enum irk_option)."""
        self._check(lib().irk_set_option(self._ctx, key, val))

    def get_option(self, key: int) -> int:
        """irk_get_option: an IRK_OPT_* value or an IRK_INFO_* fact about the last call."""
        out = np.zeros(1, dtype=np.int64)
        self._check(lib().irk_get_option(self._ctx, key, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        return int(out[0])

    def local_energy_error(self, workspace, stream=None):
        """Per-trajectory Delta H^loc_max of the last call (IRK_OPT_LOCAL_ENERGY)."""
        import torch
        _need(workspace, "workspace", torch.uint8, min_numel=self.workspace_bytes)
        out = torch.empty(self.batch, dtype=torch.float64, device=workspace.device)
        s = torch.cuda.current_stream(workspace.device) if stream is None else stream
        self._check(lib().irk_local_energy_error(self._ctx, _ptr(workspace), _ptr(out),
                                                 ctypes.c_void_p(s.cuda_stream)))
        return out

    def hist_view(self, workspace):
        """The history block of a workspace as a float64 (8, dim, batch) tensor view."""
        import torch
        nb = 8 * self.local_dim * self.batch * 8
        return workspace[64:64 + nb].view(torch.float64).view(8, self.local_dim, self.batch)


def probe_dfma(out, blocks: int, iters: int, stream) -> int:
    """Enqueue the FP64 FMA throughput probe; returns its flop count."""
    n = lib().irk_probe_dfma(_ptr(out), blocks, iters, ctypes.c_void_p(stream.cuda_stream))
    if n < 0:
        raise IrkError(E_CUDA, "irk_probe_dfma launch failed")
    return int(n)


def probe_divsqrt(a, b, stream=None):
    """(fast a/b, __ddiv_rn, fast sqrt b, __dsqrt_rn, fast 1/b, __ddiv_rn(1, b)) for
    device float64 tensors a, b."""
    import torch
    n = a.numel()
    out = torch.empty((n, 6), dtype=torch.float64, device=a.device)
    s = torch.cuda.current_stream(a.device) if stream is None else stream
    if lib().irk_probe_divsqrt(_ptr(a), _ptr(b), _ptr(out), n, ctypes.c_void_p(s.cuda_stream)):
        raise IrkError(E_CUDA, "irk_probe_divsqrt failed")
    return out


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for Integrator.set_comm (call on rank 0, broadcast)."""
    buf = ctypes.create_string_buffer(128)
    rc = lib().irk_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p))
    if rc:
        raise IrkError(rc, "irk_nccl_unique_id failed (NCCL not loadable?)")
    return buf.raw
