"""B200-native randomized K-FAC hot path (arXiv 2206.15397) behind the reference's operator API.

Host side of the drop-in boundary.  The reference is C++ (``/root/reference/proj/include/rkfac``); its operator
API is mirrored here name for name over the C-ABI in ``include/rkfac_b200.h`` (``librkfac_b200.so``, sm_100a):

=========================================================  ==================================================
reference (kfactor.hpp / rnla.hpp / optimizer.hpp)          this module
=========================================================  ==================================================
``EAKFactor``, ``ea_update(f, m)`` (kfactor.hpp:17-41)      ``EAKFactor``, ``ea_update(f, m)``
``SketchParams``, ``RngState`` (rnla.hpp:26, rng.hpp:25)    ``SketchParams``, ``RngState``
``srevd(x, p, rng)`` / ``rsvd_psd(x, p, rng)``              ``srevd`` / ``rsvd_psd`` -> ``LowRankEig``
``apply_lowrank_damped_inverse(lr, lam, v, side)``          ``apply_lowrank_damped_inverse``
``preconditioned_step`` layer loop (optimizer.hpp:139)      ``BatchedStep`` (all factors in single launches)
exceptions (errors.hpp:8-34)                                ``DimensionMismatch``, ``DampingNonpositive``, ...
=========================================================  ==================================================

Tensors are CUDA ``torch.float32`` (PyTorch is plumbing here: device memory and streams).  There is no CPU
fallback: if the library or an sm_100 device is missing, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from enum import Enum
from typing import Optional, Sequence

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librkfac_b200.so")
# A multi-group step runs on 2 streams per group (+ copy streams): with the driver's default of 8 hardware work queues
# streams share queues and serialise falsely.  Read when the CUDA context is created, so it is set at import (a host
# that already set it keeps its value); the library enables its side-stream overlap only when it sees >= 16.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

# ---------------------------------------------------------------------------------------------- errors


class RkfacError(RuntimeError):
    status = -1


class DimensionMismatch(RkfacError):  # errors.hpp:8
    status = 1


class RankDeficient(RkfacError):  # errors.hpp:12
    status = 2


class NoConvergence(RkfacError):  # errors.hpp:16
    status = 3


class DampingNonpositive(RkfacError):  # errors.hpp:20
    status = 4


class CudaError(RkfacError):
    status = 5


class NcclError(RkfacError):
    status = 6


class InvalidArgument(RkfacError):
    status = 7


_BY_STATUS = {c.status: c for c in (DimensionMismatch, RankDeficient, NoConvergence, DampingNonpositive, CudaError,
                                    NcclError, InvalidArgument)}

# ----------------------------------------------------------------------------------------- C-ABI binding

_c_i64 = C.c_int64
_c_u64 = C.c_uint64
_vp = C.c_void_p


class _FactorDesc(C.Structure):
    _fields_ = [("dim", _c_i64), ("rank", _c_i64), ("oversampling", _c_i64), ("power_iters", _c_i64)]


_lib = None

#: every entry point of include/rkfac_b200.h, with (restype, argtypes)
SIGNATURES = {
    "rkfac_create": (C.c_int, [C.POINTER(_vp), C.c_int, _vp]),
    "rkfac_destroy": (C.c_int, [_vp]),
    "rkfac_set_stream": (C.c_int, [_vp, _vp]),
    "rkfac_synchronize": (C.c_int, [_vp]),
    "rkfac_last_error": (C.c_char_p, [_vp]),
    "rkfac_status_string": (C.c_char_p, [C.c_int]),
    "rkfac_launch_count": (_c_u64, [_vp]),
    "rkfac_sample_gaussian": (C.c_int, [_vp, _c_u64, C.POINTER(_c_u64), _c_i64, _c_i64, _vp, _c_i64]),
    "rkfac_ea_update": (C.c_int, [_vp, _vp, _c_i64, _c_i64, _vp, _c_i64, _c_i64, _c_i64, C.c_double, C.c_double]),
    "rkfac_srevd": (C.c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_u64, C.POINTER(_c_u64), _vp,
                              _c_i64, _vp, C.POINTER(_c_i64)]),
    "rkfac_rsvd_psd": (C.c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_u64, C.POINTER(_c_u64), _vp,
                                 _c_i64, _vp, C.POINTER(_c_i64)]),
    "rkfac_apply_lowrank_damped_inverse": (C.c_int, [_vp, _vp, _c_i64, _vp, _c_i64, _c_i64, C.c_double, _vp,
                                                     _c_i64, _c_i64, _c_i64, C.c_int, _vp, _c_i64]),
    "rkfac_plan_create": (C.c_int, [_vp, C.POINTER(_FactorDesc), C.c_int, C.c_int, C.POINTER(_vp)]),
    "rkfac_plan_destroy": (C.c_int, [_vp]),
    "rkfac_plan_rank": (_c_i64, [_vp, C.c_int]),
    "rkfac_plan_bind_factors": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp)]),
    "rkfac_plan_bind_factors_ld": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_c_i64), C.POINTER(_vp),
                                             C.POINTER(_c_i64), C.POINTER(_vp)]),
    "rkfac_plan_bind_samples": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_c_i64)]),
    "rkfac_plan_bind_layers": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(_vp),
                                         C.POINTER(_vp), C.POINTER(_vp)]),
    "rkfac_plan_set_tags": (C.c_int, [_vp, C.POINTER(_c_u64)]),
    "rkfac_plan_ea_update": (C.c_int, [_vp, C.c_double, C.c_double]),
    "rkfac_plan_decompose": (C.c_int, [_vp, _c_u64, _c_u64]),
    "rkfac_plan_ea_decompose": (C.c_int, [_vp, C.c_double, C.c_double, _c_u64, _c_u64]),
    "rkfac_plan_set_step_seed": (C.c_int, [_vp, _c_u64, _c_u64]),
    "rkfac_plan_set_overlap": (C.c_int, [_vp, C.c_int]),
    "rkfac_plan_precondition": (C.c_int, [_vp, C.c_double]),
    "rkfac_plan_step": (C.c_int, [_vp, C.c_double, C.c_double, _c_u64, _c_u64, C.c_double]),
    "rkfac_plan_timing": (C.c_int, [_vp, C.POINTER(C.c_float), C.POINTER(C.c_int)]),
    "rkfac_plan_set_timing": (C.c_int, [_vp, C.c_int]),
    "rkfac_plan_set_ea_lo_mode": (C.c_int, [_vp, C.c_int]),
    "rkfac_plan_set_max_ctas": (C.c_int, [_vp, C.c_int]),
    "rkfac_plan_prepare": (C.c_int, [_vp, C.c_double, C.c_double, C.c_double]),
    "rkfac_plan_workspace_size": (C.c_size_t, [_vp]),
    "rkfac_sym_eig": (C.c_int, [_vp, _vp, _c_i64, _c_i64, _vp, _c_i64, _vp, _vp]),
    "rkfac_rsvd": (C.c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_u64, C.POINTER(_c_u64),
                             _vp, _c_i64, _vp, _vp, _c_i64, C.POINTER(_c_i64)]),
    "rkfac_conv_patches": (C.c_int, [_vp, _vp] + [_c_i64] * 12 + [C.c_int, C.c_double, _vp, _c_i64]),
    "rkfac_conv_grads": (C.c_int, [_vp, _vp, _c_i64, _c_i64, _c_i64, _c_i64, C.c_double, _vp, _c_i64]),
    "rkfac_nccl_unique_id": (C.c_int, [_vp]),
    "rkfac_nccl_init": (C.c_int, [_vp, _vp, C.c_int, C.c_int]),
    "rkfac_set_nccl_comm": (C.c_int, [_vp, _vp, C.c_int, C.c_int]),
    "rkfac_allgather": (C.c_int, [_vp, _vp, _vp, _c_i64]),
    "rkfac_plan_set_gather": (C.c_int, [_vp, _c_i64, C.POINTER(_c_i64), _vp]),
    "rkfac_plan_gather": (C.c_int, [_vp]),
}


def load_library(path: str = LIB_PATH):
    """Loads librkfac_b200.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run `python -m paper_2206_15397_b200.build` (no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def _check(status: int, ctx=None, what: str = ""):
    if status != 0:
        lib = load_library()
        msg = lib.rkfac_last_error(ctx).decode() if lib.rkfac_last_error(ctx) else ""
        raise _BY_STATUS.get(status, RkfacError)(f"{what}: {lib.rkfac_status_string(status).decode()}: {msg}")


# --------------------------------------------------------------------------------------------- context

_contexts: dict = {}


def _torch():
    import torch  # plumbing: device memory + streams

    return torch


class Context:
    """One C-ABI context per (device); follows torch's current stream at each call."""

    def __init__(self, device: int = 0):
        torch = _torch()
        lib = load_library()
        if not torch.cuda.is_available():
            raise CudaError("rkfac_b200 needs a CUDA device (sm_100); there is no CPU fallback")
        self.device = device
        h = _vp()
        _check(lib.rkfac_create(C.byref(h), device, _vp(torch.cuda.current_stream(device).cuda_stream)), None,
               "rkfac_create")
        self.h = h
        self.lib = lib

    def sync_stream(self):
        torch = _torch()
        _check(self.lib.rkfac_set_stream(self.h, _vp(torch.cuda.current_stream(self.device).cuda_stream)), self.h,
               "rkfac_set_stream")

    def launches(self) -> int:
        return int(self.lib.rkfac_launch_count(self.h))

    # -- multi-GPU: the NCCL communicator of the one all-gather (rkfac_nccl_init / rkfac_allgather)
    def nccl_init(self, unique_id: bytes, nranks: int, rank: int):
        """Joins the clique (blocks until every rank joined); the context owns the communicator."""
        buf = C.create_string_buffer(bytes(unique_id), len(unique_id))
        _check(self.lib.rkfac_nccl_init(self.h, C.cast(buf, _vp), nranks, rank), self.h, "nccl_init")
        self.nranks, self.rank = nranks, rank

    def allgather(self, send, recv):
        """recv (nranks * send.numel() floats, rank-major) <- every rank's send, on torch's current stream."""
        self.sync_stream()
        if recv.numel() != send.numel() * getattr(self, "nranks", 1):
            raise InvalidArgument("allgather: recv must hold nranks * send.numel() floats")
        _check(self.lib.rkfac_allgather(self.h, _ptr(send), _ptr(recv), send.numel()), self.h, "allgather")

    def __del__(self):
        try:
            self.lib.rkfac_destroy(self.h)
        except Exception:
            pass


def context(device: Optional[int] = None) -> Context:
    torch = _torch()
    load_library()
    if not torch.cuda.is_available():
        raise CudaError("rkfac_b200 needs a CUDA device (sm_100); there is no CPU fallback")
    dev = torch.cuda.current_device() if device is None else device
    if dev not in _contexts:
        _contexts[dev] = Context(dev)
    ctx = _contexts[dev]
    ctx.sync_stream()
    return ctx


def _ptr(t) -> _vp:
    return _vp(t.data_ptr())


def nccl_unique_id() -> bytes:
    """A new clique's 128-byte ncclUniqueId (rank 0 creates it and ships it to the others, e.g. by
    torch.distributed.broadcast_object_list)."""
    lib = load_library()
    buf = C.create_string_buffer(128)
    _check(lib.rkfac_nccl_unique_id(C.cast(buf, _vp)), None, "nccl_unique_id")
    return buf.raw


def _need_cuda_f32(t, name: str):
    torch = _torch()
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32):
        raise InvalidArgument(f"{name} must be a CUDA float32 tensor")
    if t.dim() != 2 or t.stride(1) != 1:
        raise InvalidArgument(f"{name} must be a row-major 2-D tensor")


# ----------------------------------------------------------------------------------- reference types


class DecompMethod(Enum):  # rnla.hpp:14
    RSVD = 0
    SREVD = 1
    EXACT = 2


class ApplySide(Enum):  # kfactor.hpp:128
    LEFT = 0
    RIGHT = 1


@dataclass
class SketchParams:  # rnla.hpp:26-30
    target_rank: int = 1
    oversampling: int = 0
    power_iters: int = 0


@dataclass
class RngState:  # rng.hpp:25-56 (seed/counter only; draws happen on the device)
    seed: int = 0
    counter: int = 0

    def substream(self, a: int, b: int = 0) -> "RngState":
        return RngState(substream_seed(self.seed, a, b))


def splitmix64(x: int) -> int:  # rng.hpp:13-18
    m = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & m
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & m
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & m
    return x ^ (x >> 31)


def substream_seed(seed: int, a: int, b: int = 0) -> int:  # rng.hpp:32-36
    return splitmix64(seed ^ splitmix64(a ^ splitmix64(b)))


@dataclass
class LowRankEig:  # rnla.hpp:17-24: u (d x r, orthonormal columns), d (r, descending)
    u: object
    d: object
    method: DecompMethod = DecompMethod.RSVD

    def rank(self) -> int:
        return int(self.d.shape[0])

    def dim(self) -> int:
        return int(self.u.shape[0])


@dataclass
class EAKFactor:  # kfactor.hpp:17-31
    mbar: object
    rho: float = 0.95
    steps: int = 0

    @staticmethod
    def create(dim: int, rho: float, zero_init: bool = False, device=None) -> "EAKFactor":
        torch = _torch()
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        m = torch.zeros(dim, dim, device=dev) if zero_init else torch.eye(dim, device=dev)
        return EAKFactor(m, rho)

    def dim(self) -> int:
        return int(self.mbar.shape[0])


# ------------------------------------------------------------------------------------------ operators


def sample_gaussian(rng: RngState, m: int, n: int, device=None):
    """rng.hpp:59-63: m x n N(0,1) draws on the device (FP64 math, FP32 store); advances rng.counter."""
    torch = _torch()
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    out = torch.empty(m, n, device=dev, dtype=torch.float32)
    ctx = context(out.device.index)
    ctr = _c_u64(rng.counter)
    _check(ctx.lib.rkfac_sample_gaussian(ctx.h, _c_u64(rng.seed), C.byref(ctr), m, n, _ptr(out), n), ctx.h,
           "sample_gaussian")
    rng.counter = int(ctr.value)
    return out


def ea_update(f: EAKFactor, m, scale: float = 1.0) -> None:
    """kfactor.hpp:33-41: f.mbar <- rho f.mbar + (1-rho) scale^2 m m^T (in place on the device)."""
    _need_cuda_f32(f.mbar, "mbar")
    _need_cuda_f32(m, "m")
    ctx = context(f.mbar.device.index)
    _check(ctx.lib.rkfac_ea_update(ctx.h, _ptr(f.mbar), f.mbar.stride(0), f.dim(), _ptr(m), m.stride(0),
                                   m.shape[0], m.shape[1], float(f.rho), float(scale)), ctx.h, "ea_update")
    f.steps += 1


def _decompose(fn_name: str, method: DecompMethod, x, params: SketchParams, rng: RngState) -> LowRankEig:
    torch = _torch()
    _need_cuda_f32(x, "x")
    if x.shape[0] != x.shape[1]:
        raise DimensionMismatch(f"{fn_name}: factor must be square")
    d = x.shape[0]
    r_cl = min(params.target_rank, d)
    ctx = context(x.device.index)
    u = torch.empty(d, max(1, r_cl), device=x.device, dtype=torch.float32)
    dv = torch.empty(max(1, r_cl), device=x.device, dtype=torch.float32)
    ctr = _c_u64(rng.counter)
    rank = _c_i64(0)
    fn = getattr(ctx.lib, fn_name)
    _check(fn(ctx.h, _ptr(x), x.stride(0), d, params.target_rank, params.oversampling, params.power_iters,
              _c_u64(rng.seed), C.byref(ctr), _ptr(u), u.stride(0), _ptr(dv), C.byref(rank)), ctx.h, fn_name)
    rng.counter = int(ctr.value)
    rr = int(rank.value)
    return LowRankEig(u[:, :rr], dv[:rr], method)


@dataclass
class SvdResult:  # eig.hpp:239-241 / rnla.hpp:62-77: u (rows x r), s (r, descending), v (cols x r)
    u: object
    s: object
    v: object


def rsvd(x, params: SketchParams, rng: RngState) -> SvdResult:
    """rnla.hpp:62-77 on a general (rows x cols) matrix; advances rng.counter by 2*cols*w like sample_gaussian."""
    torch = _torch()
    _need_cuda_f32(x, "x")
    rows, cols = x.shape
    dim = min(rows, cols)
    r_cl = min(params.target_rank, dim)
    ctx = context(x.device.index)
    u = torch.empty(rows, max(1, r_cl), device=x.device, dtype=torch.float32)
    s = torch.empty(max(1, r_cl), device=x.device, dtype=torch.float32)
    v = torch.empty(cols, max(1, r_cl), device=x.device, dtype=torch.float32)
    ctr = _c_u64(rng.counter)
    rank = _c_i64(0)
    _check(ctx.lib.rkfac_rsvd(ctx.h, _ptr(x), x.stride(0), rows, cols, params.target_rank, params.oversampling,
                              params.power_iters, _c_u64(rng.seed), C.byref(ctr), _ptr(u), u.stride(0), _ptr(s), _ptr(v),
                              v.stride(0), C.byref(rank)), ctx.h, "rsvd")
    rng.counter = int(ctr.value)
    rr = int(rank.value)
    return SvdResult(u[:, :rr], s[:rr], v[:, :rr])


def srevd(x, params: SketchParams, rng: RngState) -> LowRankEig:
    """rnla.hpp:90-105 (advances rng.counter by 2*d*w like sample_gaussian)."""
    return _decompose("rkfac_srevd", DecompMethod.SREVD, x, params, rng)


def rsvd_psd(x, params: SketchParams, rng: RngState) -> LowRankEig:
    """rnla.hpp:81-85 (V-side basis)."""
    return _decompose("rkfac_rsvd_psd", DecompMethod.RSVD, x, params, rng)


def apply_lowrank_damped_inverse(lr: LowRankEig, lam: float, v, side: ApplySide):
    """kfactor.hpp:134-161: LEFT (U D U^T + lam I)^{-1} V, RIGHT V (U D U^T + lam I)^{-1}."""
    torch = _torch()
    if lam <= 0.0:
        raise DampingNonpositive("apply_lowrank_damped_inverse: lambda must be > 0")
    _need_cuda_f32(v, "v")
    u = lr.u.contiguous() if lr.u.stride(1) != 1 else lr.u
    _need_cuda_f32(u, "u")
    dv = lr.d.contiguous()
    out = torch.empty_like(v, memory_format=torch.contiguous_format)
    ctx = context(v.device.index)
    _check(ctx.lib.rkfac_apply_lowrank_damped_inverse(ctx.h, _ptr(u), u.stride(0), _ptr(dv), lr.dim(), lr.rank(),
                                                      float(lam), _ptr(v), v.stride(0), v.shape[0], v.shape[1],
                                                      side.value, _ptr(out), out.stride(0)), ctx.h,
           "apply_lowrank_damped_inverse")
    return out


# ------------------------------------------------------------------------ exact K-FAC comparator
@dataclass
class SymEigResult:  # eig.hpp:20-25: p (n x n, eigenvectors as columns), d (n, descending)
    p: object
    d: object


def sym_eig(s, fp64: bool = False) -> SymEigResult:
    """eig.hpp:210-237 for the exact K-FAC comparator (the cubic baseline of harness.hpp:402-478 bench-inverse) and
    the spectrum snapshots: full symmetric eigendecomposition, eigenvalues descending, eigenvectors as the columns of
    ``p``.  This repo's own FP64 solver (csrc/symeig.cu: blocked Householder tridiagonalisation, divide and conquer,
    WY back-transformation) through ``rkfac_sym_eig``.  Asymmetry above 1e-4 * max(1, ||S||_max) (eig.hpp:213-215's
    1e-8 scaled for FP32 storage) raises DimensionMismatch; the symmetrised matrix is decomposed.  ``fp64`` is kept
    for call compatibility: the solver always computes in FP64."""
    torch = _torch()
    _need_cuda_f32(s, "s")
    if s.dim() != 2 or s.shape[0] != s.shape[1]:
        raise DimensionMismatch("sym_eig: matrix must be square")
    n = s.shape[0]
    p = torch.empty(n, n, device=s.device, dtype=torch.float32)
    d = torch.empty(n, device=s.device, dtype=torch.float32)
    ctx = context(s.device.index)
    _check(ctx.lib.rkfac_sym_eig(ctx.h, _ptr(s), s.stride(0), n, _ptr(p), p.stride(0), _ptr(d), None), ctx.h,
           "sym_eig")
    return SymEigResult(p, d)


def sym_eigvals(s):
    """The eigenvalues alone, descending, in FP64 (kfactor.hpp:56-63 spectrum): the same solver, no P output."""
    torch = _torch()
    _need_cuda_f32(s, "s")
    if s.dim() != 2 or s.shape[0] != s.shape[1]:
        raise DimensionMismatch("sym_eig: matrix must be square")
    n = s.shape[0]
    d = torch.empty(n, device=s.device, dtype=torch.float64)
    ctx = context(s.device.index)
    _check(ctx.lib.rkfac_sym_eig(ctx.h, _ptr(s), s.stride(0), n, None, n, None, _ptr(d)), ctx.h, "sym_eig")
    return d


def apply_eig_damped_inverse(eig: SymEigResult, lam: float, v, side: ApplySide):
    """kfactor.hpp:165-186: LEFT U (D + lam I)^{-1} U^T V, RIGHT V U (D + lam I)^{-1} U^T -- through the hot path's
    own apply kernels: Eq. 11 with a complete orthonormal U is exactly (U D U^T + lam I)^{-1}."""
    return apply_lowrank_damped_inverse(LowRankEig(eig.p, eig.d, DecompMethod.EXACT), lam, v, side)


# ------------------------------------------------------------------------------------- batched step


@dataclass
class LayerSpec:
    """One K-FAC layer: A-factor dimension (d_in+1) and G-factor dimension (d_out) (network.hpp:51-80)."""

    dim_a: int
    dim_g: int


@dataclass
class BatchedStep:
    """The batched preconditioned step (optimizer.hpp:139-167) for a fixed list of layers.

    Factor ``2l`` is layer l's A-factor and ``2l+1`` its G-factor, so the decomposition seed of factor f is
    ``RngState(root).substream(step, f)`` exactly as optimizer.hpp:189/202.  All tensors are allocated on the
    device once; ``step()`` runs EA update -> rand-EVD of every factor -> preconditioning of every layer with one
    launch per stage.
    """

    layers: Sequence[LayerSpec]
    rank: int = 220
    oversampling: int = 10
    power_iters: int = 4
    method: DecompMethod = DecompMethod.SREVD
    n_samples: Sequence[int] = ()
    device: int = 0
    factor_indices: Optional[Sequence[int]] = None  # global factor tags (multi-GPU shards keep global seeds)
    max_ctas: int = 0  # cap of the persistent tensor-core grids (0: all SMs; StreamedStep leaves SMs to other groups)
    factors: list = field(default_factory=list, init=False)
    bases_t: list = field(default_factory=list, init=False)
    dvals: list = field(default_factory=list, init=False)
    samples: list = field(default_factory=list, init=False)
    grads: list = field(default_factory=list, init=False)
    outs: list = field(default_factory=list, init=False)
    mids: list = field(default_factory=list, init=False)

    def __post_init__(self):
        torch = _torch()
        self.ctx = context(self.device)
        lib = self.ctx.lib
        dims = []
        for L in self.layers:
            dims += [L.dim_a, L.dim_g]
        self.dims = dims
        descs = (_FactorDesc * len(dims))(*[_FactorDesc(d, self.rank, self.oversampling, self.power_iters)
                                           for d in dims])
        h = _vp()
        meth = 1 if self.method == DecompMethod.SREVD else 0
        _check(lib.rkfac_plan_create(self.ctx.h, descs, len(dims), meth, C.byref(h)), self.ctx.h, "plan_create")
        self.h = h
        if self.max_ctas:
            _check(lib.rkfac_plan_set_max_ctas(h, int(self.max_ctas)), self.ctx.h, "set_max_ctas")
        dev = torch.device("cuda", self.device)
        self.ranks = [int(lib.rkfac_plan_rank(h, f)) for f in range(len(dims))]
        lds = []
        for f, d in enumerate(dims):
            # factors live in row-pitch-padded storage (pitch multiple of 32 floats) so the EA update and the
            # X*Q products feed them to TMA directly; self.factors[f] is the d x d view
            ld = (d + 31) // 32 * 32
            lds.append(ld)
            self.factors.append(torch.zeros(d, ld, device=dev)[:, :d])
            self.bases_t.append(torch.zeros(self.ranks[f], d, device=dev))
            self.dvals.append(torch.zeros(self.ranks[f], device=dev))
        arr = lambda ts: (_vp * len(ts))(*[t.data_ptr() for t in ts])  # noqa: E731
        ldf = (_c_i64 * len(dims))(*lds)
        _check(lib.rkfac_plan_bind_factors_ld(h, arr(self.factors), ldf, arr(self.bases_t), None, arr(self.dvals)),
               self.ctx.h, "bind_factors")
        if self.factor_indices is not None:
            tags = (_c_u64 * len(dims))(*[int(t) for t in self.factor_indices])
            _check(lib.rkfac_plan_set_tags(h, tags), self.ctx.h, "set_tags")
        if self.n_samples:
            ns = list(self.n_samples)
            if len(ns) == 1:
                ns = ns * len(dims)
            for f, d in enumerate(dims):
                self.samples.append(torch.zeros(d, ns[f], device=dev))
            nn = (_c_i64 * len(dims))(*ns)
            _check(lib.rkfac_plan_bind_samples(h, arr(self.samples), nn), self.ctx.h, "bind_samples")
        nl = len(self.layers)
        for L in self.layers:
            self.grads.append(torch.zeros(L.dim_g, L.dim_a, device=dev))
            self.outs.append(torch.zeros(L.dim_g, L.dim_a, device=dev))
            self.mids.append(torch.zeros(L.dim_g, L.dim_a, device=dev))
        a_idx = (C.c_int * nl)(*[2 * l for l in range(nl)])
        g_idx = (C.c_int * nl)(*[2 * l + 1 for l in range(nl)])
        _check(lib.rkfac_plan_bind_layers(h, nl, a_idx, g_idx, arr(self.grads), arr(self.outs), arr(self.mids)),
               self.ctx.h, "bind_layers")

    # stages
    def ea_update(self, rho: float = 0.95, scale: float = 1.0):
        self.ctx.sync_stream()
        _check(self.ctx.lib.rkfac_plan_ea_update(self.h, rho, scale), self.ctx.h, "plan_ea_update")

    def decompose(self, rng_root: int, step: int):
        self.ctx.sync_stream()
        _check(self.ctx.lib.rkfac_plan_decompose(self.h, _c_u64(rng_root), _c_u64(step)), self.ctx.h,
               "plan_decompose")

    def ea_decompose(self, rng_root: int, step: int, rho: float = 0.95, scale: float = 1.0):
        """ea_update + decompose of the same step (Omega generated next to the EA update; bitwise the two calls)."""
        self.ctx.sync_stream()
        _check(self.ctx.lib.rkfac_plan_ea_decompose(self.h, rho, scale, _c_u64(rng_root), _c_u64(step)), self.ctx.h,
               "plan_ea_decompose")

    def precondition(self, lam: float):
        if lam <= 0.0:
            raise DampingNonpositive("apply_lowrank_damped_inverse: lambda must be > 0")
        self.ctx.sync_stream()
        _check(self.ctx.lib.rkfac_plan_precondition(self.h, lam), self.ctx.h, "plan_precondition")

    def step(self, rng_root: int, step: int, lam: float, rho: float = 0.95, scale: float = 1.0):
        if lam <= 0.0:
            raise DampingNonpositive("apply_lowrank_damped_inverse: lambda must be > 0")
        self.ctx.sync_stream()
        _check(self.ctx.lib.rkfac_plan_step(self.h, rho, scale, _c_u64(rng_root), _c_u64(step), lam), self.ctx.h,
               "plan_step")

    def set_overlap(self, on: bool):
        """Overlapped power iteration (rkfac_plan_set_overlap; off by default): shorter per-factor latency chain,
        tail Ritz values perturbed by ~(6e-8 lambda_1 / lambda_r)^2 -- see :func:`overlap_error_estimate`."""
        _check(self.ctx.lib.rkfac_plan_set_overlap(self.h, 1 if on else 0), self.ctx.h, "plan_set_overlap")

    def set_step_seed(self, rng_root: int, step: int):
        """(rng_root, step) of the next replay of a CUDA graph captured from this plan's step / decomposition."""
        _check(self.ctx.lib.rkfac_plan_set_step_seed(self.h, _c_u64(rng_root), _c_u64(step)), self.ctx.h,
               "plan_set_step_seed")

    def prepare(self, lam: float, rho: float = 0.95, scale: float = 1.0):
        """Build every stage step(lam, rho, scale) uses, without launching (so the step can be graph-captured)."""
        if lam <= 0.0:
            raise DampingNonpositive("apply_lowrank_damped_inverse: lambda must be > 0")
        _check(self.ctx.lib.rkfac_plan_prepare(self.h, rho, scale, lam), self.ctx.h, "plan_prepare")

    def set_timing(self, on: bool):
        _check(self.ctx.lib.rkfac_plan_set_timing(self.h, 1 if on else 0), self.ctx.h, "set_timing")

    def set_gather(self, chunk: int, offsets: Sequence[int], gathered):
        """step() ends with the all-gather (rkfac_plan_set_gather): layer l's output packed at offsets[l] of this
        rank's chunk; every rank's chunk lands in ``gathered`` (nranks * chunk floats).  ``gathered=None`` disables."""
        offs = (_c_i64 * len(self.layers))(*[int(o) for o in offsets])
        _check(self.ctx.lib.rkfac_plan_set_gather(self.h, int(chunk), offs, _ptr(gathered) if gathered is not None
                                                  else None), self.ctx.h, "set_gather")

    def gather(self):
        self.ctx.sync_stream()
        _check(self.ctx.lib.rkfac_plan_gather(self.h), self.ctx.h, "gather")

    def workspace_bytes(self) -> int:
        return int(self.ctx.lib.rkfac_plan_workspace_size(self.h))

    def set_ea_lo_mode(self, mode: int):
        """EA operands' TF32 lo planes: -1 automatic, 0 formed in shared memory, 1 stored by a split pass."""
        _check(self.ctx.lib.rkfac_plan_set_ea_lo_mode(self.h, int(mode)), self.ctx.h, "set_ea_lo_mode")

    TIMING_KINDS = ("ea", "decompose", "precondition", "xq_gemm", "orth", "eig", "step")

    def timing(self):
        """{stage: (total ms, count)} since set_timing(True); call after torch.cuda.synchronize()."""
        sums = (C.c_float * 7)()
        cnts = (C.c_int * 7)()
        _check(self.ctx.lib.rkfac_plan_timing(self.h, sums, cnts), self.ctx.h, "timing")
        return {k: (float(sums[i]), int(cnts[i])) for i, k in enumerate(self.TIMING_KINDS)}

    def lowrank(self, f: int) -> LowRankEig:
        meth = self.method if self.method != DecompMethod.EXACT else DecompMethod.SREVD
        return LowRankEig(self.bases_t[f].t(), self.dvals[f], meth)

    def __del__(self):
        try:
            self.ctx.lib.rkfac_plan_destroy(self.h)
        except Exception:
            pass


STREAMED_TC_CTAS = 132


def overlap_error_estimate(dvals) -> float:
    """Predicted relative perturbation of the last retained Ritz value under the overlapped power iteration
    (``set_overlap``): (2^-24 * lambda_1 / lambda_r)^2, from the eigenvalues of a previous decomposition of the factor
    (K-FAC spectra move slowly between T_KI refreshes).  Enable the overlap while this stays below the parity bar."""
    d = dvals.detach().double().cpu() if hasattr(dvals, "detach") else dvals
    top, last = float(d[0]), float(d[len(d) - 1])
    if last <= 0.0:
        return float("inf")
    return (2.0 ** -24 * top / last) ** 2


def _replay_with_seed(g, rng_root, step):
    """The pinned (root, step) pair is read by a copy node of the replay, asynchronously: a NEW pair may only be
    written once the previous replay has consumed the old one, so a change of seed first waits for the event recorded
    behind the previous replay (free when, as in training, other work separates two K-FAC steps)."""
    torch = _torch()
    if rng_root is not None and (rng_root, step) != getattr(g, "_seed", None):
        ev = getattr(g, "_last", None)
        if ev is not None:
            ev.synchronize()
        g.step_obj.set_step_seed(rng_root, step)
        g._seed = (rng_root, step)
    g.graph.replay()
    if getattr(g, "_last", None) is None:
        g._last = torch.cuda.Event()
    g._last.record(torch.cuda.current_stream(g.step_obj.device))


class StepGraph:
    """One full preconditioned step (EA -> rand-EVD -> precondition of every layer, every group's stream) captured
    once as a CUDA graph and replayed: ~70 dependent launches per group chain are submitted as one graph launch, so the
    inter-kernel gaps and the host enqueue cost leave the step.  Stages are built by ``prepare`` first (capture only
    enqueues kernels); the Omega seeds (rng_root, step) are read at replay time (``replay(rng_root, step)``), so one
    graph serves every step of a training run.  Replays read the current contents of the step's device buffers
    (factors, samples, grads) and are bitwise identical to ``step_obj.step``.
    """

    def __init__(self, step_obj, rng_root: int, step: int, lam: float, rho: float = 0.95, scale: float = 1.0):
        torch = _torch()
        self.step_obj = step_obj
        step_obj.prepare(lam, rho, scale)
        dev = step_obj.device
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        n0 = step_obj.ctx.launches()
        with torch.cuda.stream(s):
            with torch.cuda.graph(self.graph, stream=s):
                step_obj.step(rng_root, step, lam, rho, scale)
        torch.cuda.current_stream(dev).wait_stream(s)
        self.launches = step_obj.ctx.launches() - n0  # kernels per replay

    def replay(self, rng_root: Optional[int] = None, step: Optional[int] = None):
        """Replay the captured step; (rng_root, step), when given, select this replay's Omega substreams (the captured
        step reads them from a pinned host pair: rkfac_plan_set_step_seed), else the pair of the last replay."""
        _replay_with_seed(self, rng_root, step)


class HostStepGraph:
    """``StreamedStep.step_host`` -- the step from pinned host inputs to pinned host outputs, copies included --
    captured once as one CUDA graph and replayed: the ~100 host-side enqueues of a step (copies and ~70 launches per
    group) leave the critical path, so every group's samples land and its chain starts at once instead of behind the
    previous group's enqueue.  Replays read the current contents of the pinned host buffers given at capture (the
    staging buffers a training loop refills each step) and write the host outputs; bitwise ``step_host``."""

    def __init__(self, step_obj, rng_root: int, step: int, lam: float, h_samples, h_grads, h_outs, rho: float = 0.95,
                 scale: float = 1.0):
        torch = _torch()
        self.step_obj = step_obj
        step_obj.prepare(lam, rho, scale)
        dev = step_obj.device
        step_obj.step_host(rng_root, step, lam, h_samples, h_grads, h_outs, rho, scale)  # streams/events created
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        n0 = step_obj.ctx.launches()
        with torch.cuda.stream(s):
            with torch.cuda.graph(self.graph, stream=s):
                step_obj.step_host(rng_root, step, lam, h_samples, h_grads, h_outs, rho, scale)
        torch.cuda.current_stream(dev).wait_stream(s)
        self.launches = step_obj.ctx.launches() - n0

    def replay(self, rng_root: Optional[int] = None, step: Optional[int] = None):
        _replay_with_seed(self, rng_root, step)


class StreamedStep:
    """The batched step split into ``groups`` independent layer groups, each a :class:`BatchedStep` (its own plan)
    run on its own CUDA stream and joined back into the caller's stream.

    The per-factor kernels of the decomposition are latency-bound on a few SMs (Cholesky-inverse: one CTA per factor,
    the tridiagonalisation: one 4-CTA cluster per factor); running a second group's tensor-core stages meanwhile
    fills the idle SMs.  Groups are formed by LPT on the decomposition cost, exactly like the multi-GPU shards, and
    factor tags stay global, so every result is bitwise identical to the single-plan step.  Public surface (factors,
    samples, grads, outs, lowrank, stages) mirrors BatchedStep in the original layer order.
    """

    def __init__(self, layers: Sequence[LayerSpec], groups: int = 2, rank: int = 220, oversampling: int = 10,
                 power_iters: int = 4, method: DecompMethod = DecompMethod.SREVD, n_samples: Sequence[int] = (),
                 device: int = 0, factor_indices: Optional[Sequence[int]] = None, max_ctas: Optional[int] = None):
        from .partition import layer_cost, lpt_partition

        torch = _torch()
        self.layers = list(layers)
        self.device = device
        self.method = method
        nl = len(self.layers)
        tags = list(factor_indices) if factor_indices is not None else list(range(2 * nl))
        costs = [layer_cost(L.dim_a, L.dim_g, rank, oversampling) for L in self.layers]
        self.parts = [p for p in lpt_partition(costs, max(1, min(groups, nl))) if p]
        if max_ctas is None:
            # a persistent tensor-core grid on every SM would keep the other groups' latency-bound kernels (Cholesky-
            # inverse, tridiagonalisation clusters) waiting; 132 of 148 measured best for 2 VGG16 groups
            # (with more groups each grid gets a smaller share: 2 x 148 / groups, between 64 and 132 -- measured with
            # 5 VGG16 groups: 148 / 132 / 100 / 64 / 48 CTAs -> 7.02 / 7.01 / 6.96 / 6.93 / 6.95 ms)
            g = len(self.parts)
            max_ctas = max(64, min(STREAMED_TC_CTAS, (2 * 148 // g) & ~1)) if g > 1 else 0
        ns = list(n_samples)
        self.subs = []
        for part in self.parts:
            sub_ns = ns if len(ns) <= 1 else [ns[2 * l + w] for l in part for w in (0, 1)]
            self.subs.append(BatchedStep([self.layers[l] for l in part], rank=rank, oversampling=oversampling,
                                         power_iters=power_iters, method=method, n_samples=sub_ns, device=device,
                                         factor_indices=[tags[2 * l + w] for l in part for w in (0, 1)],
                                         max_ctas=max_ctas))
        self.ctx = self.subs[0].ctx
        # the group with the most decomposition work is the critical chain: its stream gets the highest priority so
        # its kernels take SMs first when other groups' grids drain (RKFAC_STREAM_PRIORITY=0 disables)
        gcost = [sum(costs[l] for l in part) for part in self.parts]
        lo_pri, hi_pri = torch.cuda.Stream.priority_range()
        use_pri = os.environ.get("RKFAC_STREAM_PRIORITY", "1") != "0"
        order = sorted(range(len(self.parts)), key=lambda g: -gcost[g])
        pri = [0] * len(self.parts)
        if use_pri and len(self.parts) > 1:
            graded = os.environ.get("RKFAC_STREAM_PRIORITY", "1") == "2"
            for rank_, g in enumerate(order):
                pri[g] = max(hi_pri, hi_pri + rank_) if graded else (hi_pri if rank_ == 0 else 0)
                if pri[g] > lo_pri:
                    pri[g] = lo_pri
        self.streams = [torch.cuda.Stream(device=device, priority=pri[g]) for g in range(len(self.subs))]
        self._issue_order = order
        # views in the original order
        self.dims, self.factors, self.samples, self.bases_t, self.dvals, self.ranks = [], [], [], [], [], []
        self.grads, self.outs, self.mids = [None] * nl, [None] * nl, [None] * nl
        self._owner = [None] * (2 * nl)
        for s, (part, sub) in enumerate(zip(self.parts, self.subs)):
            for i, l in enumerate(part):
                self.grads[l], self.outs[l], self.mids[l] = sub.grads[i], sub.outs[i], sub.mids[i]
                for w in (0, 1):
                    self._owner[2 * l + w] = (s, 2 * i + w)
        for f in range(2 * nl):
            s, j = self._owner[f]
            sub = self.subs[s]
            self.dims.append(sub.dims[j])
            self.factors.append(sub.factors[j])
            self.samples.append(sub.samples[j] if sub.samples else None)
            self.bases_t.append(sub.bases_t[j])
            self.dvals.append(sub.dvals[j])
            self.ranks.append(sub.ranks[j])

    def _fan_out(self, fn):
        torch = _torch()
        main = torch.cuda.current_stream(self.device)
        fork = torch.cuda.Event()
        fork.record(main)
        joins = []
        for sub, st in zip(self.subs, self.streams):
            st.wait_event(fork)
            with torch.cuda.stream(st):
                fn(sub)
                ev = torch.cuda.Event()
                ev.record(st)
                joins.append(ev)
        for ev in joins:
            main.wait_event(ev)
        self.ctx.sync_stream()

    def ea_update(self, rho: float = 0.95, scale: float = 1.0):
        self._fan_out(lambda s: s.ea_update(rho, scale))

    def decompose(self, rng_root: int, step: int):
        self._fan_out(lambda s: s.decompose(rng_root, step))

    def precondition(self, lam: float):
        if lam <= 0.0:
            raise DampingNonpositive("apply_lowrank_damped_inverse: lambda must be > 0")
        self._fan_out(lambda s: s.precondition(lam))

    def step(self, rng_root: int, step: int, lam: float, rho: float = 0.95, scale: float = 1.0):
        if lam <= 0.0:
            raise DampingNonpositive("apply_lowrank_damped_inverse: lambda must be > 0")
        self._fan_out(lambda s: s.step(rng_root, step, lam, rho, scale))

    def prepare(self, lam: float, rho: float = 0.95, scale: float = 1.0):
        for sub in self.subs:
            sub.prepare(lam, rho, scale)

    def set_step_seed(self, rng_root: int, step: int):
        for sub in self.subs:
            sub.set_step_seed(rng_root, step)

    def set_overlap(self, on: bool):
        for sub in self.subs:
            sub.set_overlap(on)

    def step_host(self, rng_root: int, step: int, lam: float, h_samples, h_grads, h_outs, rho: float = 0.95,
                  scale: float = 1.0, timeline: Optional[list] = None):
        """The step with its inputs and outputs in (pinned) host memory, in the original factor / layer order.

        Per group, on the group's stream: H2D of its samples -> EA -> rand-EVD; meanwhile a copy stream brings its
        gradients (needed only by the preconditioning); then precondition -> D2H of its results.  One group's copies
        overlap the other groups' kernels, and every gradient upload overlaps its own group's decomposition.
        ``timeline`` (a list) receives, per group, timing events (samples in, decomposed, preconditioned, results out)
        and the fork event first, for tools/e2e_timeline.py.
        """
        if lam <= 0.0:
            raise DampingNonpositive("apply_lowrank_damped_inverse: lambda must be > 0")
        torch = _torch()
        if not hasattr(self, "_copy_streams"):
            self._copy_streams = [torch.cuda.Stream(device=self.device) for _ in self.subs]
        main = torch.cuda.current_stream(self.device)
        timed = timeline is not None
        fork = torch.cuda.Event(enable_timing=timed)
        fork.record(main)
        if timed:
            timeline.append(("fork", fork))

        def mark(st, name, g):
            if timed:
                e = torch.cuda.Event(enable_timing=True)
                e.record(st)
                timeline.append((f"group{g}:{name}", e))

        # 1. every group's samples first (the host-to-device engine serves copies in submission order: a group's
        #    gradients, needed only at the end of its chain, must not delay the next group's samples), each group's
        #    EA + rand-EVD enqueued right behind its own samples
        last_samples = None
        for g in self._issue_order:  # the critical group's uploads first
            sub, st, part = self.subs[g], self.streams[g], self.parts[g]
            st.wait_event(fork)
            with torch.cuda.stream(st):
                for i, l in enumerate(part):
                    for w in (0, 1):
                        if sub.samples:
                            sub.samples[2 * i + w].copy_(h_samples[2 * l + w], non_blocking=True)
                last_samples = torch.cuda.Event()
                last_samples.record(st)
                mark(st, "samples_in", g)
                if sub.samples:
                    sub.ea_decompose(rng_root, step, rho, scale)
                else:
                    sub.decompose(rng_root, step)
                mark(st, "decomposed", g)
        # 2. the gradients, behind all the samples on the copy engine
        got_grads = {}
        for g in self._issue_order:
            sub, cp, part = self.subs[g], self._copy_streams[g], self.parts[g]
            cp.wait_event(last_samples)
            with torch.cuda.stream(cp):
                for i, l in enumerate(part):
                    sub.grads[i].copy_(h_grads[l], non_blocking=True)
                got_grads[g] = torch.cuda.Event()
                got_grads[g].record(cp)
        # 3. per group: precondition -> results to the host
        joins = []
        for g in self._issue_order:
            sub, st, part = self.subs[g], self.streams[g], self.parts[g]
            with torch.cuda.stream(st):
                st.wait_event(got_grads[g])
                sub.precondition(lam)
                mark(st, "preconditioned", g)
                for i, l in enumerate(part):
                    h_outs[l].copy_(sub.outs[i], non_blocking=True)
                mark(st, "results_out", g)
                ev = torch.cuda.Event()
                ev.record(st)
                joins.append(ev)
        for ev in joins:
            main.wait_event(ev)
        self.ctx.sync_stream()

    def lowrank(self, f: int) -> LowRankEig:
        s, j = self._owner[f]
        return self.subs[s].lowrank(j)
