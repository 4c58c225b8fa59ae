"""K-FAC optimizer orchestration around the batched GPU step: factor statistics, the
decomposition cache on the T_KI schedule and the hyper-parameter schedules of the reference optimizer.

Host logic only -- every FLOP runs in the batched plan (:class:`BatchedStep`): EA updates, rand-EVDs and the
preconditioning of all layers per launch.  Mirrors optimizer.hpp:25-220 and network.hpp:155-165:

* :func:`run_schedules` is optimizer.hpp:67-90 (T_KI, lambda, alpha, target rank and oversampling by epoch, with the
  same ConfigError checks), :func:`needs_recompute` is optimizer.hpp:118-121;
* :func:`factor_statistics` forms the per-layer A matrices (activations with the ones row, network.hpp:88-91) and
  the G matrices (back-propagated signals), :meth:`KfacOptimizer.accumulate_factors` is network.hpp:155-165
  (EA update with M = X / sqrt(n));
* :meth:`KfacOptimizer.step` is optimizer.hpp:139-167: refresh the cached decompositions of every layer when the
  schedule says so (step % T_KI == 0, or the method changed), then S_l = LEFT_Gamma(RIGHT_A(J_l)) for all layers.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum
from typing import List, Optional, Sequence


class ConfigError(ValueError):  # errors.hpp ConfigError
    pass


class Method(Enum):  # optimizer.hpp Method
    KFAC = 0
    RS_KFAC = 1
    SRE_KFAC = 2


@dataclass
class ScheduleOverrides:  # optimizer.hpp:30-36
    lam: Optional[float] = None
    alpha: Optional[float] = None
    target_rank: Optional[int] = None
    oversampling: Optional[int] = None
    t_ki: Optional[int] = None


@dataclass
class OptimizerConfig:  # optimizer.hpp:38-53
    method: Method = Method.KFAC  # the reference default (optimizer.hpp:39)
    rho: float = 0.95
    t_ku: int = 10        # factor-update period
    n_pwr_it: int = 4     # sketch power iterations
    n_bs: int = 256       # batch size
    weight_decay: float = 7e-4
    overrides: ScheduleOverrides = field(default_factory=ScheduleOverrides)

    def validate(self):
        if self.t_ku < 1:
            raise ConfigError("OptimizerConfig: T_KU must be >= 1")
        if not (0.0 < self.rho < 1.0):
            raise ConfigError("OptimizerConfig: rho must be in (0,1)")


@dataclass
class ResolvedSchedule:  # optimizer.hpp:55-61
    alpha: float = 0.3
    lam: float = 0.1
    target_rank: int = 220
    oversampling: int = 10
    t_ki: int = 50


def _ind(epoch: int, at: int) -> float:
    return 1.0 if epoch >= at else 0.0


def run_schedules(cfg: OptimizerConfig, epoch: int) -> ResolvedSchedule:
    """optimizer.hpp:67-90 (the paper's section 5 schedules)."""
    o = cfg.overrides
    s = ResolvedSchedule()
    s.t_ki = o.t_ki if o.t_ki is not None else int(50 - 20 * _ind(epoch, 20))
    s.lam = o.lam if o.lam is not None else 0.1 - 0.05 * _ind(epoch, 25) - 0.04 * _ind(epoch, 35)
    s.alpha = (o.alpha if o.alpha is not None else
               0.3 - 0.1 * _ind(epoch, 2) - 0.1 * _ind(epoch, 3) - 0.07 * _ind(epoch, 13) - 0.02 * _ind(epoch, 18)
               - 0.007 * _ind(epoch, 27) - 0.002 * _ind(epoch, 40))
    s.target_rank = o.target_rank if o.target_rank is not None else int(220 + 10 * _ind(epoch, 15))
    s.oversampling = (o.oversampling if o.oversampling is not None else
                      int(10 + _ind(epoch, 22) + _ind(epoch, 30)))
    if s.t_ki < cfg.t_ku:
        raise ConfigError("schedule: T_KI must be >= T_KU")
    if s.lam <= 0.0:
        raise ConfigError("schedule: lambda must be > 0")
    return s


def needs_recompute(cached_method, step: int, t_ki: int, want) -> bool:
    """optimizer.hpp:118-121."""
    return cached_method is None or cached_method != want or step % t_ki == 0


def factor_statistics(activations: Sequence, deltas: Sequence):
    """Per-layer (A, G) matrices of one batch (network.hpp:82-130): A_l = [a_{l-1}; 1] ((d_in+1) x n, the ones row
    of with_ones_row) and G_l = delta_l (d_out x n).  Inputs are device tensors with samples as columns."""
    import torch

    a_mats = [torch.cat([a, torch.ones(1, a.shape[1], device=a.device, dtype=a.dtype)], 0) for a in activations]
    return a_mats, list(deltas)


def _pair(v):
    return (int(v), int(v)) if isinstance(v, int) else (int(v[0]), int(v[1]))


def conv_output_size(h: int, w: int, kernel_size, stride=1, padding=0, dilation=1):
    (kh, kw), (sh, sw), (ph, pw), (dh, dw) = map(_pair, (kernel_size, stride, padding, dilation))
    return (h + 2 * ph - dh * (kh - 1) - 1) // sh + 1, (w + 2 * pw - dw * (kw - 1) - 1) // sw + 1


def conv_factor_statistics(x, dy, kernel_size, stride=1, padding=0, dilation=1, out_a=None, out_g=None):
    """The EA operands of one convolution layer (the conv analogue of network.hpp:88-95, 134 and 155-165), on the GPU
    (csrc/stats.cu through rkfac_conv_patches / rkfac_conv_grads):

    * A = patch matrix of x (B x C x H x W) with a ones row: (C*kh*kw + 1) x n, n = B*Ho*Wo;
    * G = output gradient dy (B x Co x Ho x Wo) as Co x n;

    both already scaled by 1/sqrt(n) (accumulate_factors' M = X / sqrt(n)), so the plan's EA runs with scale 1.
    ``out_a`` / ``out_g`` (row-major, contiguous) may be the plan's sample buffers (no extra copy)."""
    import torch

    from . import InvalidArgument, _check, _ptr, context

    for t, nm in ((x, "x"), (dy, "dy")):
        if not (t.is_cuda and t.dtype == torch.float32 and t.dim() == 4 and t.is_contiguous()):
            raise InvalidArgument(f"conv_factor_statistics: {nm} must be a contiguous CUDA float32 NCHW tensor")
    (kh, kw), (sh, sw), (ph, pw), (dh, dw) = map(_pair, (kernel_size, stride, padding, dilation))
    B, Cin, H, W = x.shape
    Ho, Wo = conv_output_size(H, W, (kh, kw), (sh, sw), (ph, pw), (dh, dw))
    if dy.shape[0] != B or dy.shape[2] != Ho or dy.shape[3] != Wo:
        from . import DimensionMismatch

        raise DimensionMismatch("conv_factor_statistics: dy does not match the convolution's output shape")
    n = B * Ho * Wo
    d_a, d_g = Cin * kh * kw + 1, dy.shape[1]
    a = out_a if out_a is not None else torch.empty(d_a, n, device=x.device)
    g = out_g if out_g is not None else torch.empty(d_g, n, device=x.device)
    if tuple(a.shape) != (d_a, n) or tuple(g.shape) != (d_g, n) or a.stride(1) != 1 or g.stride(1) != 1:
        raise InvalidArgument("conv_factor_statistics: output buffers must be (C*kh*kw+1) x n and Co x n, row-major")
    scale = 1.0 / math.sqrt(n)
    ctx = context(x.device.index)
    _check(ctx.lib.rkfac_conv_patches(ctx.h, _ptr(x), B, Cin, H, W, kh, kw, sh, sw, ph, pw, dh, dw, 1, scale,
                                      _ptr(a), a.stride(0)), ctx.h, "conv_patches")
    _check(ctx.lib.rkfac_conv_grads(ctx.h, _ptr(dy), B, d_g, Ho, Wo, scale, _ptr(g), g.stride(0)), ctx.h,
           "conv_grads")
    return a, g


@dataclass
class StepTimings:  # optimizer.hpp:92-96 (device time, CUDA events)
    factor_update: float = 0.0
    decomposition: float = 0.0
    inverse_apply: float = 0.0


class KfacOptimizer:
    """The preconditioner of RS-KFAC / SRE-KFAC / K-FAC for a fixed list of layers on one GPU.

    ``layers``: :class:`LayerSpec` list (dim_a = d_in + 1, dim_g = d_out); ``rng_seed``: the optimizer's RngState
    seed (decomposition of factor 2l+which at step k draws Omega from substream(k, 2l+which), optimizer.hpp:189).
    Factors start as the identity (kfactor.hpp:27) unless ``zero_init``.
    """

    def __init__(self, layers: Sequence, cfg: OptimizerConfig, n_samples: int, rng_seed: int = 0, device: int = 0,
                 zero_init: bool = False):
        cfg.validate()
        self.layers = list(layers)
        self.cfg = cfg
        self.n = n_samples
        self.rng_seed = rng_seed
        self.device = device
        self.zero_init = zero_init
        self._plan = None
        self._plan_key = None
        self._cached_method = None
        self._exact = None  # per-factor SymEigResult (K-FAC)
        self.timings = StepTimings()

    # -- plan (rebuilt only when the schedule changes the sketch size)
    def _ensure_plan(self, sch: ResolvedSchedule):
        import torch

        from . import BatchedStep, DecompMethod

        meth = DecompMethod.RSVD if self.cfg.method == Method.RS_KFAC else DecompMethod.SREVD
        key = (sch.target_rank, sch.oversampling, meth)
        if self._plan_key == key:
            return
        old = self._plan
        self._plan = BatchedStep(self.layers, rank=sch.target_rank, oversampling=sch.oversampling,
                                 power_iters=self.cfg.n_pwr_it, method=meth, n_samples=[self.n], device=self.device)
        for f, x in enumerate(self._plan.factors):
            if old is not None:
                x.copy_(old.factors[f])  # the EA state carries over
            elif not self.zero_init:
                x.copy_(torch.eye(x.shape[0], device=x.device))
        self._plan_key = key
        self._cached_method = None  # a new plan holds no decomposition

    @property
    def plan(self):
        return self._plan

    def accumulate_factors(self, a_mats: Sequence, g_mats: Sequence, epoch: int = 0):
        """network.hpp:155-165: EA update of every factor with M = X / sqrt(n) (all factors in one launch)."""
        import torch

        if len(a_mats) != len(self.layers) or len(g_mats) != len(self.layers):
            from . import DimensionMismatch

            raise DimensionMismatch("accumulate_factors: per-layer matrix count")
        self._ensure_plan(run_schedules(self.cfg, epoch))
        p = self._plan
        for l, (a, g) in enumerate(zip(a_mats, g_mats)):
            if a.shape[1] != self.n or g.shape[1] != self.n:
                from . import DimensionMismatch

                raise DimensionMismatch("accumulate_factors: batch size differs from the plan's n")
            p.samples[2 * l].copy_(a)
            p.samples[2 * l + 1].copy_(g)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p.ea_update(self.cfg.rho, 1.0 / math.sqrt(self.n))
        e1.record()
        e1.synchronize()
        self.timings.factor_update += e0.elapsed_time(e1) / 1e3

    def step(self, gradients: Sequence, step: int, epoch: int = 0) -> List:
        """optimizer.hpp:139-167: preconditioned updates S_l (d_out x (d_in+1)) of every layer."""
        import torch

        from . import ApplySide, DecompMethod, apply_eig_damped_inverse, sym_eig

        sch = run_schedules(self.cfg, epoch)
        self._ensure_plan(sch)
        p = self._plan
        want = {Method.KFAC: DecompMethod.EXACT, Method.RS_KFAC: DecompMethod.RSVD,
                Method.SRE_KFAC: DecompMethod.SREVD}[self.cfg.method]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        if needs_recompute(self._cached_method, step, sch.t_ki, want):
            if want == DecompMethod.EXACT:
                self._exact = [sym_eig(x.contiguous(), fp64=True) for x in p.factors]  # comparator accuracy
            else:
                p.decompose(self.rng_seed, step)
            self._cached_method = want
        ev[1].record()
        for l, g in enumerate(gradients):
            p.grads[l].copy_(g)
        if want == DecompMethod.EXACT:
            outs = []
            for l in range(len(self.layers)):
                m = apply_eig_damped_inverse(self._exact[2 * l], sch.lam, p.grads[l], ApplySide.RIGHT)
                outs.append(apply_eig_damped_inverse(self._exact[2 * l + 1], sch.lam, m, ApplySide.LEFT))
        else:
            p.precondition(sch.lam)
            outs = [o.clone() for o in p.outs]
        ev[2].record()
        ev[2].synchronize()
        self.timings.decomposition += ev[0].elapsed_time(ev[1]) / 1e3
        self.timings.inverse_apply += ev[1].elapsed_time(ev[2]) / 1e3
        return outs


# ------------------------------------------------------------------ spectrum snapshots and run logs (8(f) #4)
@dataclass
class SpectrumReport:  # kfactor.hpp:44-54
    eigenvalues: list          # decreasing, clamped at 0
    lambda_max: float = 0.0

    def count_above(self, epsilon: float) -> int:
        thr = epsilon * self.lambda_max
        return sum(1 for v in self.eigenvalues if v >= thr)


def spectrum(factor) -> SpectrumReport:
    """kfactor.hpp:56-63 on a device factor: full eigenvalues (this repo's FP64 eigensolver, csrc/symeig.cu, on the
    FP32 factor), clamped at 0."""
    from . import sym_eigvals

    d = sym_eigvals(factor.contiguous()).cpu().tolist()
    ev = [max(0.0, v) for v in d]
    return SpectrumReport(ev, ev[0] if ev else 0.0)


@dataclass
class SpectrumSnapshot:  # harness.hpp:65-69
    step: int
    layer: int
    eigenvalues: list


@dataclass
class StepRecord:  # harness.hpp (run log row)
    step: int
    epoch: int
    loss: float
    acc: float
    timings: StepTimings


def snapshot_a_factors(opt: "KfacOptimizer", step: int) -> List[SpectrumSnapshot]:
    """harness.hpp:214-218: the forward (A) factor spectrum of every layer."""
    return [SpectrumSnapshot(step, l, spectrum(opt.plan.factors[2 * l]).eigenvalues) for l in range(len(opt.layers))]


def _fmt(v: float) -> str:  # harness.hpp:239-243 ("%.17g")
    return "%.17g" % v


def write_runlog_csv(path: str, steps: Sequence[StepRecord]):
    """harness.hpp:276-285: step,epoch,loss,acc,t_factor,t_decomp,t_apply."""
    with open(path, "w") as f:
        f.write("step,epoch,loss,acc,t_factor,t_decomp,t_apply\n")
        for r in steps:
            f.write(f"{r.step},{r.epoch},{_fmt(r.loss)},{_fmt(r.acc)},{_fmt(r.timings.factor_update)},"
                    f"{_fmt(r.timings.decomposition)},{_fmt(r.timings.inverse_apply)}\n")


def write_spectrum_csv(path: str, snapshots: Sequence[SpectrumSnapshot]):
    """harness.hpp:287-293: step,layer,idx,eigenvalue."""
    with open(path, "w") as f:
        f.write("step,layer,idx,eigenvalue\n")
        for s in snapshots:
            for i, v in enumerate(s.eigenvalues):
                f.write(f"{s.step},{s.layer},{i},{_fmt(v)}\n")


def decay_orders(eigenvalues: Sequence[float], modes: int) -> float:
    """harness.hpp:307-315: log10(lambda_1 / lambda_m) over the first `modes` eigenvalues."""
    if not eigenvalues:
        return 0.0
    m = min(modes, len(eigenvalues))
    head, tail = eigenvalues[0], eigenvalues[m - 1]
    if head <= 0.0:
        return 0.0
    if tail <= 0.0:
        return 300.0
    return math.log10(head / tail)
