#!/usr/bin/env python
"""bench.py -- the randomized K-FAC hot path (EA update -> rand-EVD of every factor -> damped low-rank
preconditioning of every layer gradient) on the BASELINE config-3 workload: the VGG16_bn-shaped full step
(32 factors, 16 layers, n=128, r=min(220,d), p=10, q=4, lambda=0.1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload vgg16|wide4096|wide16384]

Our arm: one process per GPU (torchrun for N>1), layers LPT-sharded across ranks, one NCCL all-gather of the
preconditioned gradients.  A step = one EA update of every factor + rand-EVD of every factor + preconditioning of
every layer (+ the all-gather).  value = factors inverted per second of whole step (all ranks) = 32 / step time.
Reference arm (--impl reference): the reference's own C++ CPU code (oracle/_ref, the unmodified headers compiled
with the reference's own flags) on all of the box's host cores, one factor per std::thread: every timed step is the
WHOLE step of the workload, measured (config 5 alone -- hours per FP64 step -- is a proxy, extrapolated and labelled
in `cpu_baseline.sample`).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "K-factor rand-EVD inversions/s and precond-step ms; % of TF32/HBM roofline"
UNIT = "inversions/s"
ROOT_SEED = 220615397  # synthetic factor statistics
OMEGA_ROOT = 7
GRAD_ROOT = 99
# dram__bytes_read.sum + dram__bytes_write.sum of one X*Q launch of THIS workload, from that workload's own ncu --set
# full capture (profiles/); None for a workload not captured yet
XQ_TRAFFIC = {"vgg16": 606247680 + 29901312}  # X read once; its lo plane is formed in smem
XQ_TRAFFIC_SRC = {"vgg16": "profiles/r02_xq_full.txt (dram__bytes_read.sum + dram__bytes_write.sum; CTA-pair kernel)"}

VGG_A = [28, 577, 577, 1153, 1153, 2305, 2305, 2305, 4609, 4609, 4609, 4609, 4609, 513, 513, 513]
VGG_G = [64, 64, 128, 128, 256, 256, 256, 512, 512, 512, 512, 512, 512, 512, 512, 10]

WORKLOADS = {
    # name: (layers [(dA, dG)], n, e, rank, p, q, lambda, ea warm-up steps)
    "vgg16": ([(a, g) for a, g in zip(VGG_A, VGG_G)], 128, 1.0, 220, 10, 4, 0.1, 20),
    "wide4096": ([(4096, 4096)], 128, 0.8, 220, 10, 4, 0.1, 50),
    "wide16384": ([(16384, 16384)] * 4, 512, 1.2, 256, 16, 4, 0.05, 10),
}


def sketch_width(d, r, p):
    return d if r > d else min(r + p, d)


def work_model(layers, n, r, p, q):
    """Algorithmic work per factor / layer."""
    fac = []
    for a, g in layers:
        for d in (a, g):
            w = sketch_width(d, r, p)
            rr = min(r, d)
            f_gemm = (2 * q + 2) * 2.0 * d * d * w + 2.0 * d * w * w + 2.0 * d * w * rr
            f_orth = 6.0 * (2 * q + 1) * d * w * w
            f_ea = 2.0 * n * d * d
            b_ea = 8.0 * d * d + 4.0 * n * d
            b_gemm = (2 * q + 2) * 4.0 * d * d
            fac.append(dict(d=d, w=w, r=rr, f_gemm=f_gemm, f_orth=f_orth, f_ea=f_ea, b_ea=b_ea, b_gemm=b_gemm,
                            f_xq_launch=2.0 * d * d * w))
    lay = []
    for i, (a, g) in enumerate(layers):
        ra, rg = min(r, a), min(r, g)
        wa, wg = sketch_width(a, r, p), sketch_width(g, r, p)
        lay.append(dict(f_ap=4.0 * g * a * (ra + rg), b_ap=8.0 * g * a + 4.0 * (a * wa + g * wg)))
    return fac, lay


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, device_index=0, period=0.02):  # the timed region is ~0.1 s: several samples under load
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period
        self.dev = device_index
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.dev)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        return self

    def _run(self):
        nv = self.nv
        names = {
            getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksThrottleReasonSwPowerCap", 0x4): "sw_power_cap",
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, nm in names.items():
                    if mask & bit:
                        self.reasons.add(nm)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# -------------------------------------------------------------------------------------- CPU baseline
def _cpu_lib():
    """The reference's own code compiled with its own flags (oracle/_ref/librkfac_ref_stock.so, CMakeLists.txt:9);
    the parity build, then the restatement, only when that is absent (the kind says which)."""
    import oracle

    if oracle.ref_stock_available():
        return oracle.ref_stock(), "reference", "oracle/_ref/librkfac_ref_stock.so (-O3 -march=native -funroll-loops)"
    if oracle.ref_available():
        return oracle.ref(), "reference", "oracle/_ref/librkfac_ref.so (-O3 -march=x86-64-v3 -ffp-contract=off)"
    return oracle.port(), "port", "oracle/liboracle.so (C restatement)"


class CpuStep:
    """The reference's whole step on the same workload, MEASURED (no extrapolation): one EA update of every factor,
    srevd of every factor (Omega from RngState(7).substream(0, f)), RIGHT_A then LEFT_G of every layer
    (optimizer.hpp:139-167), one factor (then one layer) per std::thread over `threads` host cores (ref_step_threaded;
    the functions are pure).  Inputs are built once, untimed: the factors after the workload's
    EA warm-up (FP64, zero init, the synthetic statistics of SURVEY.md 8(d)), the timed step's samples and the
    gradients, all from the reference RNG."""

    def __init__(self, layers, n, e, r, p, q, lam, warm, threads=None):
        import numpy as np

        import oracle

        self.lib, self.kind, self.build = _cpu_lib()
        port = oracle.port()
        self.layers, self.n, self.r, self.p, self.q, self.lam = layers, n, r, p, q, lam
        self.threads = threads or os.cpu_count() or 1
        dims = [d for a, g in layers for d in (a, g)]

        def warm_factor(f):  # zero-init EA over `warm` steps in FP64 (numpy: kfactor.hpp:33-41 restated)
            d = dims[f]
            x = np.zeros((d, d))
            for k in range(warm):
                m = port.synthetic_m(ROOT_SEED, k, f, n, d, e)
                x *= 0.95
                x += 0.05 * (m @ m.T)
                x = 0.5 * (x + x.T)
            return x

        self.factors0 = oracle.parallel_map(warm_factor, range(len(dims)), min(4, self.threads))
        self.ms = [port.synthetic_m(ROOT_SEED, warm, f, n, d, e) for f, d in enumerate(dims)]
        self.grads = [port.sample_gaussian(port.substream(GRAD_ROOT, l, 0), 0, g, a)[0] for l, (a, g) in
                      enumerate(layers)]
        self.outs = [np.zeros((g, a)) for a, g in layers]

    def run(self, threads=None):
        """One timed step (s) on `threads` cores; returns (seconds, per-phase seconds)."""
        facs = [x.copy() for x in self.factors0]  # the EA updates in place: every step starts from the same state
        nth = threads or self.threads
        t0 = time.perf_counter()
        ph = self.lib.step_threaded("srevd", nth, [a for a, _ in self.layers], [g for _, g in self.layers], facs,
                                    self.ms, [self.n] * len(self.ms), 0.95, self.r, self.p, self.q, OMEGA_ROOT, 0,
                                    self.lam, self.grads, self.outs)
        return time.perf_counter() - t0, [float(x) for x in ph]


def cpu_reference_sample(layers, n, e, r, p, q, lam, budget_s, threads=None):
    """Config 5 only (d = 16384: the reference's FP64 step takes hours): the reference's own code on a proxy of the
    workload, on `threads` host cores, extrapolated (`cpu_baseline.sample` says so).

    The sample is the smallest layers (by decomposition cost) whose estimated makespan fits `budget_s`; the full
    step time is extrapolated as kappa * LPT-makespan(full) with kappa = measured / modelled sample time, the
    model being the algorithmic flops of SURVEY.md 8(d) at a rate calibrated on the sample itself."""
    import numpy as np

    import oracle

    ref = _cpu_lib()[0]
    port = oracle.port()
    cores = threads or os.cpu_count() or 1
    fac, lay = work_model(layers, n, r, p, q)
    cost_f = [f["f_gemm"] + f["f_orth"] + f["f_ea"] for f in fac]
    cost_l = [cost_f[2 * i] + cost_f[2 * i + 1] + lay[i]["f_ap"] for i in range(len(layers))]
    rate = 3.5e9  # flop/s per core, SURVEY.md 6 (refined after the run)

    def lpt_makespan(costs, nthreads):
        loads = [0.0] * max(1, nthreads)
        for c in sorted(costs, reverse=True):
            k = loads.index(min(loads))
            loads[k] += c
        return max(loads)

    order = sorted(range(len(layers)), key=lambda i: cost_l[i])
    chosen = []
    for i in order:
        trial = chosen + [i]
        fcost = [cost_f[2 * j + w] for j in trial for w in (0, 1)]
        if lpt_makespan(fcost, cores) / rate > budget_s and chosen:
            break
        chosen = trial
    chosen.sort()
    # very wide factors (config 5: d = 16384, hours per factor in FP64): even the smallest layer exceeds the budget,
    # so the sample is a proxy layer of the same shape family, both dims scaled down (sketch unchanged) until its
    # modelled time fits; the calibration kappa is then measured on the proxy
    proxy = None
    i0 = chosen[0]
    if lpt_makespan([cost_f[2 * i0], cost_f[2 * i0 + 1]], cores) / rate > 2.0 * budget_s:
        a0, g0 = layers[i0]
        sc = 1.0
        while sc > 0.02:
            pa, pg = max(2 * (r + p), int(a0 * sc)), max(2 * (r + p), int(g0 * sc))
            pf, _ = work_model([(pa, pg)], n, r, p, q)
            if lpt_makespan([x["f_gemm"] + x["f_orth"] + x["f_ea"] for x in pf], cores) / rate <= budget_s:
                break
            sc *= 0.85
        proxy = (pa, pg)
        layers = list(layers)
        full_cost_f = cost_f
        layers[i0] = proxy
        fac_p, lay_p = work_model([proxy], n, r, p, q)
        cost_f = list(cost_f)
        cost_f[2 * i0] = fac_p[0]["f_gemm"] + fac_p[0]["f_orth"] + fac_p[0]["f_ea"]
        cost_f[2 * i0 + 1] = fac_p[1]["f_gemm"] + fac_p[1]["f_orth"] + fac_p[1]["f_ea"]
        chosen = [i0]
    sub = [layers[i] for i in chosen]
    # inputs in FP64 (zero-init EA from the same synthetic stream as the GPU run; untimed)
    dims_a = [a for a, _ in sub]
    dims_g = [g for _, g in sub]
    factors, ms, ns = [], [], []
    for j, li in enumerate(chosen):
        for which, d in enumerate((layers[li][0], layers[li][1])):
            f = 2 * li + which
            x = np.zeros((d, d))
            ms.append(port.synthetic_m(ROOT_SEED, 0, f, n, d, e))  # one EA update per factor in the timed step
            factors.append(x)
            ns.append(n)
    grads, outs = [], []
    for li in chosen:
        a, g = layers[li]
        jm, _ = port.sample_gaussian(port.substream(GRAD_ROOT, li, 0), 0, g, a)
        grads.append(jm)
        outs.append(np.zeros((g, a)))
    # warm the factors with a few EA updates so the decomposition sees a non-trivial spectrum (untimed)
    for k in range(1, 3):
        for idx, (li, which) in enumerate([(li, w) for li in chosen for w in (0, 1)]):
            d = layers[li][which]
            factors[idx] = port.ea_update(factors[idx], port.synthetic_m(ROOT_SEED, k, 2 * li + which, n, d, e), 0.95)
    nth = min(cores, 2 * len(chosen))
    t0 = time.perf_counter()
    if hasattr(ref, "step_threaded"):
        ph = ref.step_threaded("srevd", nth, dims_a, dims_g, factors, ms, ns, 0.95, r, p, q, OMEGA_ROOT, 0, lam,
                               grads, outs)
        kind = "reference"
    else:  # restatement, threaded via ctypes (GIL released)
        kind = "port"
        ph = None
        fl = [(li, w) for li in chosen for w in (0, 1)]

        def one(idx):
            li, w = fl[idx]
            xx = port.ea_update(factors[idx], ms[idx], 0.95)
            return port.srevd(xx, r, p, q, port.substream(OMEGA_ROOT, 0, 2 * li + w), 0)

        decs = oracle.parallel_map(one, range(len(fl)), nth)
        for j in range(len(chosen)):
            port.precondition(decs[2 * j][0], decs[2 * j][1], decs[2 * j + 1][0], decs[2 * j + 1][1], lam, grads[j])
    t_sample = time.perf_counter() - t0
    sample_cost = [cost_f[2 * j + w] for j in chosen for w in (0, 1)]
    model_sample = lpt_makespan(sample_cost, nth) / rate
    kappa = t_sample / model_sample
    if proxy is not None:
        cost_f = full_cost_f
    full_time = kappa * lpt_makespan(cost_f, cores) / rate
    full_time = max(full_time, kappa * max(cost_f) / rate)
    nf = len(fac)
    what = (f"a proxy layer {proxy} of layer {i0} (all dims scaled down, same r/p/q)" if proxy is not None else
            f"layers {chosen} ({2 * len(chosen)} of {nf} factors)")
    desc = (f"reference srevd step (EA update + rand-EVD + RIGHT/LEFT apply) on {what} with {nth} threads took "
            f"{t_sample:.2f}s; whole-step time extrapolated as LPT makespan over {cores} cores of the per-factor "
            f"algorithmic work (SURVEY.md 8(d)), calibrated on the sample: {full_time:.2f}s")
    return {"value": nf / full_time, "unit": UNIT, "cores": nth, "kind": kind, "sample": desc,
            "sample_seconds": t_sample, "extrapolated_step_s": full_time,
            "phase_seconds": None if ph is None else [float(x) for x in ph]}


SINGLE_THREAD_FILE = os.path.join(ROOT, "profiles", "r02_cpu_1thread.json")


def single_thread_record(workload):
    """The reference's single-thread step on this workload, measured once on the GPU box's host by
    `python bench.py --impl reference --cpu-threads 1 --steps 1` (a ~4-minute run, too long for every bench run) and
    committed; reported next to the all-core figure with its provenance."""
    try:
        with open(SINGLE_THREAD_FILE) as fh:
            rec = json.load(fh)
        return rec if rec.get("config", {}).get("workload") == workload else None
    except Exception:
        return None


def run_reference_arm(args, wl):
    """The reference's own CPU implementation of the path (--impl reference): every timed step is the WHOLE step of
    the workload (CpuStep: EA -> 32 srevd -> 16 preconditionings), measured, on all host cores.  One untimed warm-up
    step (the CPU has nothing to JIT; it pages in the inputs); timed steps stop once 200 s of CPU time have been spent
    so the run ends within a few minutes (`steps` is the count actually timed).  Config 5 (hours per FP64 step) is
    the one workload measured on a proxy and extrapolated (cpu_reference_sample)."""
    layers, n, e, r, p, q, lam, warm = wl
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    nf = 2 * len(layers)
    threads = args.cpu_threads or os.cpu_count() or 1
    if args.workload == "wide16384":
        budget = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
        vals = []
        for i in range(1 + args.steps):
            res = cpu_reference_sample(layers, n, e, r, p, q, lam, budget, threads=threads)
            if i >= 1:
                vals.append(res["extrapolated_step_s"])
        t, timed = statistics.median(vals), len(vals)
        cpu = {k: res[k] for k in ("kind", "cores", "sample")}
    else:
        cs = CpuStep(layers, n, e, r, p, q, lam, warm, threads)
        if args.warmup > 0:
            cs.run()  # warm-up (skipped with --warmup 0, e.g. for the 4-minute single-thread record)
        vals, phases, spent = [], [], 0.0
        for i in range(args.steps):
            s, ph = cs.run()
            vals.append(s)
            phases.append(ph)
            spent += s
            if spent + s > 200.0:
                break
        t, timed = statistics.median(vals), len(vals)
        cpu = {"kind": cs.kind, "cores": threads,
               "sample": f"the whole {args.workload} step ({nf} factors: EA update + srevd + RIGHT/LEFT apply), measured "
                         f"{timed}x on {threads} host threads (one factor per std::thread); build {cs.build}; "
                         f"median phase seconds EA/srevd/apply "
                         f"{[round(statistics.median(x), 3) for x in zip(*phases)]}"}
    v = nf / t
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": timed, "steps_requested": args.steps, "warmup": min(1, args.warmup), "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "factors": nf, "layers": len(layers), "rank": r,
                       "oversampling": p, "power_iters": q, "lambda": lam, "n": n},
            "cpu_baseline": cpu | {"value": v, "unit": UNIT},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline_line(args, wl):
    """`cpu_baseline` of our arm (rank 0, N = 1): ONE measured whole step of the reference on all host cores (about 20 s
    for VGG16 on 16 cores), plus the committed single-thread measurement; config 5 uses the extrapolated proxy."""
    layers, n, e, r, p, q, lam, warm = wl
    nf = 2 * len(layers)
    threads = args.cpu_threads or os.cpu_count() or 1
    if args.workload == "wide16384":
        return cpu_reference_sample(layers, n, e, r, p, q, lam, budget_s=args.cpu_budget, threads=threads)
    cs = CpuStep(layers, n, e, r, p, q, lam, warm, threads)
    t, ph = cs.run()
    out = {"value": nf / t, "unit": UNIT, "cores": threads, "kind": cs.kind,
           "sample": f"one whole {args.workload} step ({nf} factors: EA update + srevd + RIGHT/LEFT apply), measured "
                     f"on {threads} host threads, one factor per std::thread; build {cs.build}",
           "step_seconds": t, "phase_seconds": ph}
    st = single_thread_record(args.workload)
    if st:
        out["single_thread"] = {"value": st["value"], "unit": UNIT, "step_seconds": st["ms_per_step"] / 1e3,
                                "source": os.path.relpath(SINGLE_THREAD_FILE, ROOT)}
    return out


# -------------------------------------------------------------------------------------------- our arm
def run_ours(args, wl):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2206_15397_b200 as rk
    from paper_2206_15397_b200.partition import GatherLayout, layer_cost, lpt_partition

    layers, n, e, r, p, q, lam, warm_steps = wl
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    costs = [layer_cost(a, g, r, p) for a, g in layers]
    # --emulate-world N --emulate-rank k: run rank k's shard of an N-GPU job alone on this GPU (no collective), to
    # measure every shard's critical path on a one-GPU box (tools/shard_projection.py)
    part_world, part_rank = (args.emulate_world, args.emulate_rank) if args.emulate_world else (world, rank)
    parts = lpt_partition(costs, part_world)
    mine = parts[part_rank]
    sizes = [a * g for a, g in layers]
    layout = GatherLayout.build(sizes, parts)
    shapes = [(g, a) for a, g in layers]

    specs = [rk.LayerSpec(layers[l][0], layers[l][1]) for l in mine]
    tags = [2 * l + w for l in mine for w in (0, 1)]
    step = rk.BatchedStep(specs, rank=r, oversampling=p, power_iters=q, method=rk.DecompMethod.SREVD,
                          n_samples=[n], device=local, factor_indices=tags)
    ctx = step.ctx
    inv_sqrt_n = 1.0 / math.sqrt(n)

    def fill_samples(k):
        """M_f = X^T / sqrt(n), X = Z diag(s), Z = gaussian(substream(ROOT_SEED, k, f))."""
        for i, f in enumerate(tags):
            d = step.dims[i]
            z = rk.sample_gaussian(rk.RngState(rk.substream_seed(ROOT_SEED, k, f)), n, d, device=dev)
            s = torch.arange(1, d + 1, device=dev, dtype=torch.float64).pow(-e)
            step.samples[i].copy_((z.double() * s[None, :] * inv_sqrt_n).t().float())

    # untimed warm-up of the EA statistics (zero init)
    for k in range(warm_steps):
        fill_samples(k)
        step.ea_update(0.95, 1.0)
    fill_samples(warm_steps)  # the timed step's fresh statistics
    for i, l in enumerate(mine):
        a, g = layers[l]
        j = rk.sample_gaussian(rk.RngState(rk.substream_seed(GRAD_ROOT, l, 0)), g, a, device=dev)
        step.grads[i].copy_(j)
    factors0 = [x.clone() for x in step.factors]  # every timed step starts from the same EA state
    # The timed step runs the layers as `groups` independent plans on their own streams (StreamedStep: bitwise the
    # single-plan result); the single plan `probe` is kept for the per-stage timing and the roofline of the
    # all-factor grouped launches.
    probe = step
    if args.groups > 1:
        step = rk.StreamedStep(specs, groups=args.groups, rank=r, oversampling=p, power_iters=q,
                               method=rk.DecompMethod.SREVD, n_samples=[n], device=local, factor_indices=tags)
        for dst, src in ((step.samples, probe.samples), (step.grads, probe.grads)):
            for a, b in zip(dst, src):
                a.copy_(b)
    if args.overlap:
        step.set_overlap(True)
        probe.set_overlap(True)
    torch.cuda.synchronize()

    send = torch.zeros(layout.chunk, dtype=torch.float32, device=dev)
    recv = torch.empty(world * layout.chunk, dtype=torch.float32, device=dev)
    if world > 1:
        # the collective runs through the C-ABI (rkfac_nccl_init / rkfac_allgather): torch.distributed only ships the
        # NCCL unique id and does the barriers / max-over-ranks timing
        uid = [rk.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.nccl_init(uid[0], world, rank)

    graph = None  # CUDA graph of the whole step (rk.StepGraph), captured after the eager warm-up

    def gather():
        """The one collective: pack this rank's preconditioned gradients and all-gather them over
        NVLink/NVSwitch (ncclAllGather through rkfac_allgather).  On one GPU every layer's result is already in place,
        so there is nothing to move."""
        if world == 1:
            return
        for i, l in enumerate(mine):
            send[layout.offsets[l]:layout.offsets[l] + sizes[l]].copy_(step.outs[i].view(-1))
        ctx.allgather(send, recv)

    def one_step():
        if graph is not None:
            graph.replay(OMEGA_ROOT, 0)  # the step id is a replay-time input (rkfac_plan_set_step_seed)
        else:
            step.step(OMEGA_ROOT, 0, lam, 0.95, 1.0)
        gather()

    def reset(st=None):
        for x, x0 in zip((st or step).factors, factors0):
            x.copy_(x0)

    for _ in range(args.warmup):
        reset()
        one_step()
    torch.cuda.synchronize()
    if args.graph:
        reset()
        graph = rk.StepGraph(step, OMEGA_ROOT, 0, lam, 0.95, 1.0)
        for _ in range(2):  # replays are warmed too
            reset()
            one_step()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    if args.profile_step:  # one step inside cudaProfilerStart/Stop, for `ncu --profile-from-start off`
        reset()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        one_step()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        return

    if args.trace:  # the concurrent kernel timeline of one step (CUPTI through torch.profiler) -> tools/timeline.py
        from torch.profiler import ProfilerActivity, profile

        reset()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            one_step()
            torch.cuda.synchronize()
        rows = [{"name": e.name, "ts": e.time_range.start, "dur": e.time_range.end - e.time_range.start,
                 "stream": getattr(e, "stream", None) if hasattr(e, "stream") else None}
                for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
        try:  # the chrome trace carries stream / grid per kernel
            prof.export_chrome_trace(args.trace)
        except Exception as ex:  # noqa: BLE001
            print("chrome trace failed:", ex, file=sys.stderr)
            with open(args.trace, "w") as fh:
                json.dump(rows, fh)
        return

    # ---- timed region: K steps (factor restore is outside the events) ----
    stream = torch.cuda.current_stream(dev)
    launches0 = ctx.launches()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.nvtx.range_push("timed")
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            reset()
            ev[i][0].record(stream)
            one_step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    if world > 1:
        dist.barrier()
    launches = ctx.launches() - launches0 + (graph.launches * args.steps if graph is not None else 0)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms_local = sum(step_ms) / len(step_ms)
    # per-stage timing and the roofline: the single plan (all factors per launch), K more steps, untimed above
    probe.set_timing(True)
    for _ in range(args.steps):
        reset(probe)
        probe.step(OMEGA_ROOT, 0, lam, 0.95, 1.0)
    torch.cuda.synchronize()
    timing = probe.timing()
    probe.set_timing(False)
    t = torch.tensor([ms_local], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    nf_total = 2 * len(layers)

    # ---- e2e through the public API with host buffers (pinned H2D of inputs, D2H of results) ----
    h_samples = [x.cpu().pin_memory() for x in step.samples]
    h_grads = [x.cpu().pin_memory() for x in step.grads]
    h_outs = [torch.empty_like(x, device="cpu").pin_memory() for x in step.outs]
    h2d = sum(x.numel() * 4 for x in h_samples) + sum(x.numel() * 4 for x in h_grads)
    d2h = sum(x.numel() * 4 for x in h_outs)
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]

    def e2e_step():
        if not isinstance(step, rk.StreamedStep):
            for hs, ds in zip(h_samples, step.samples):
                ds.copy_(hs, non_blocking=True)
            for hg, dg in zip(h_grads, step.grads):
                dg.copy_(hg, non_blocking=True)
            step.step(OMEGA_ROOT, 0, lam, 0.95, 1.0)
            gather()
            for ho, do in zip(h_outs, step.outs):
                ho.copy_(do, non_blocking=True)
            return
        # the public host-buffer step: per group, samples H2D -> EA -> rand-EVD while the gradients upload on a copy
        # stream, then precondition -> results D2H (one group's copies overlap the other group's kernels), replayed
        # as one CUDA graph (rk.HostStepGraph: the host enqueue of ~100 copies / launches leaves the critical path)
        if hgraph is not None:
            hgraph.replay(OMEGA_ROOT, 0)
        else:
            step.step_host(OMEGA_ROOT, 0, lam, h_samples, h_grads, h_outs, 0.95, 1.0)
        gather()

    hgraph = None
    if isinstance(step, rk.StreamedStep) and args.e2e_graph:
        reset()
        hgraph = rk.HostStepGraph(step, OMEGA_ROOT, 0, lam, h_samples, h_grads, h_outs, 0.95, 1.0)
        torch.cuda.synchronize()

    for i in range(args.warmup + args.steps):
        reset()
        if i >= args.warmup:
            e2e_ev[i - args.warmup][0].record(stream)
        e2e_step()
        if i >= args.warmup:
            e2e_ev[i - args.warmup][1].record(stream)
    torch.cuda.synchronize()
    e2e_local = sum(a.elapsed_time(b) for a, b in e2e_ev) / args.steps
    te = torch.tensor([e2e_local], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item())

    # ---- roofline of the dominant kernel (the grouped X*Q product) and per-stage fractions ----
    fac, lay = work_model(layers, n, r, p, q)
    mine_f = [fac[f] for f in tags]
    peaks, basis = load_peaks()
    xq_ms, xq_cnt = timing["xq_gemm"]
    xq_avg = xq_ms / max(1, xq_cnt)
    f_xq_launch = sum(f["f_xq_launch"] for f in mine_f)
    achieved = f_xq_launch / (xq_avg * 1e-3) / 1e12
    # 3xTF32 issues three tf32 MMAs per algorithmic FMA: its ceiling is the measured dense bf16 rate / 2 (TF32)
    # / 3.  The burst bf16 figure applies when the clock record of the timed region shows no power cap and the SM
    # clock at its maximum (the kernel then runs at the clock the burst figure was measured at); else the sustained.
    clocks = clk.summary()
    capped = ("sw_power_cap" in clocks["reasons"] or clocks["sm_mhz"] is None or clocks["sm_max_mhz"] is None
              or clocks["sm_mhz"] < 0.97 * clocks["sm_max_mhz"])
    peak_key = "bf16_tflops_sustained" if capped else "bf16_tflops"
    tf32_peak = peaks.get(peak_key, peaks["bf16_tflops"]) / 2.0
    xq_peak = tf32_peak / 3.0
    ea_ms = timing["ea"][0] / max(1, timing["ea"][1])
    ap_ms = timing["precondition"][0] / max(1, timing["precondition"][1])
    ea_bytes = sum(f["b_ea"] for f in mine_f)
    ap_bytes = sum(lay[l]["b_ap"] for l in mine)
    stages = {k: (v[0] / max(1, v[1]) if k not in ("xq_gemm", "orth") else v[0] / max(1, args.steps))
              for k, v in timing.items()}

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline and not args.emulate_world:
            try:
                cpu = cpu_baseline_line(args, wl)
            except Exception as ex:  # noqa: BLE001
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {ex}"}
        value = nf_total / (ms * 1e-3)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.workload, "factors": nf_total, "layers": len(layers), "rank": r,
                       "oversampling": p, "power_iters": q, "lambda": lam, "n": n, "method": "srevd",
                       "parallelism": f"layer-LPT x{world}" + (" + NCCL all-gather" if world > 1 else " (no collective on one GPU)"),
                       "streams_per_gpu": args.groups,
                       "cuda_graph": bool(args.graph), "overlapped_power_iteration": bool(args.overlap),
                       "l2": f"inputs ({sum(4 * d * d for a, g in layers for d in (a, g)) / 1e6:.0f} MB of factors) "
                             "exceed the 126 MB L2; no flush",
                       "value_def": "factors inverted per second of the whole step (EA + rand-EVD + precondition "
                                    "+ the all-gather on N > 1 GPUs) = factors / step time"},
            "precond_step_ms": ms,
            "stage_ms": stages,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": xq_peak, "unit": "TFLOP/s",
                         "frac": achieved / xq_peak, "traffic": XQ_TRAFFIC.get(args.workload),
                         "kernel": "tc_gemm_kernel<3>: grouped X*Q product (all factors, one launch), tcgen05 3xTF32 on "
                                   "CTA pairs (cta_group::2); fallback to single-CTA tiles when under-filled",
                         "peak_basis": f"{basis} {'sustained' if capped else 'burst'} bf16 "
                                       f"{peaks.get(peak_key, peaks['bf16_tflops'])} TF/s / 2 (TF32) / 3 (3xTF32 MMAs "
                                       f"per FMA); {'power cap or clock below max' if capped else 'no cap, max clock'}"
                                       f" in the timed region",
                         "traffic_source": XQ_TRAFFIC_SRC.get(args.workload),
                         "frac_of_tf32": achieved / tf32_peak},
            "ea_hbm": {"achieved_gbs": ea_bytes / (ea_ms * 1e-3) / 1e9, "peak_gbs": peaks["hbm_gbs"],
                       "frac": ea_bytes / (ea_ms * 1e-3) / 1e9 / peaks["hbm_gbs"]},
            "apply_hbm": {"achieved_gbs": ap_bytes / (ap_ms * 1e-3) / 1e9, "peak_gbs": peaks["hbm_gbs"],
                          "frac": ap_bytes / (ap_ms * 1e-3) / 1e9 / peaks["hbm_gbs"]},
            "e2e": {"value": nf_total / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches // max(1, args.steps),
            "gpu_launches_total": launches,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "emulated_shard": ({"world": part_world, "rank": part_rank, "layers": list(mine)} if args.emulate_world
                               else None),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="vgg16", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="config 5 proxy sample budget (s)")
    ap.add_argument("--cpu-threads", type=int, default=0, help="host threads of the CPU baseline (0: all)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--groups", type=int, default=5, help="layer groups on concurrent streams (StreamedStep; 5 gave the best e2e)")
    ap.add_argument("--profile-step", action="store_true", help="run one step under cudaProfilerStart/Stop and exit")
    ap.add_argument("--overlap", action="store_true",
                    help="opt-in overlapped power iteration (rkfac_plan_set_overlap; shortens a shard's latency chain, "
                         "parity holds while lambda_r / lambda_1 >~ 1e-5: DESIGN.md 4.1)")
    ap.add_argument("--trace", default="", help="write the kernel timeline of one step (chrome trace) and exit")
    ap.add_argument("--emulate-world", type=int, default=0, help="run one shard of an N-GPU job alone (projection)")
    ap.add_argument("--emulate-rank", type=int, default=0)
    ap.add_argument("--e2e-graph", action=argparse.BooleanOptionalAction, default=True,
                    help="replay the host-buffer e2e step as one CUDA graph (rk.HostStepGraph)")
    ap.add_argument("--graph", action=argparse.BooleanOptionalAction, default=True,
                    help="replay the timed step as one CUDA graph (rk.StepGraph: ~320 launches on 10 streams become "
                         "one graph launch; the Omega step id is a replay-time input); --no-graph times eager calls")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference_arm(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
