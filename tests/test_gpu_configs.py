"""GPU parity at BASELINE.json's full configuration sizes (configs 2, 4 and 5).

* Config 2 (d = 4096 pair, r = 220, p = 10, q = 4, lambda = 0.1): the CUDA path against the CPU oracle itself
  (oracle/rkfac_oracle.c srevd + Eq. 11, ~45 s on the host) on the same FP64 factors and the same Omega seeds.
* Config 4 (VGG16_bn step sharded over 2 / 4 / 8 GPUs): every rank's shard (LPT layer partition, global factor
  tags, partition.py) is run as its own plan on this one GPU, packed and "all-gathered" exactly as bench.py does,
  and must be BITWISE the 1-GPU step.  The ranks never wait on each other, so one GPU suffices.
* Config 5 (d = 16384, r = 256, p = 16, q = 4, lambda = 0.05): the CPU oracle would need hours, so the reference
  algorithm (rnla.hpp:47-56 randomized_range, 90-105 srevd; kfactor.hpp:134-161 Eq. 11) is restated in torch FP64
  on the GPU with the oracle's own FP64 Omega, plus the size-independent properties: orthonormal U, exact
  recovery of an exactly low-rank factor, and the Eq. 11 eigen-identity (U D U^T + lam I)^-1 u_i = u_i / (d_i+lam).
Tolerances: the north-star bar, rel. <= 1e-4 (reconstruction U L U^T, top-r eigenvalues, preconditioned gradient).
"""
import math

import numpy as np
import pytest

from tests.helpers import GRAD_ROOT, OMEGA_ROOT, ROOT_SEED, eig_err, orth_err, recon_err, rel_fro

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _t32(a, dev):
    import torch

    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32), device=dev)


def _np64(t):
    return t.detach().double().cpu().numpy()


def _orth_tol(d):
    """FP32 basis of length d: each entry of U^T U accumulates ~sqrt(d) FP32 roundings (measured 1.9e-5 at
    d = 4096), so the orthonormality bar scales with sqrt(d)."""
    return 4e-5 * math.sqrt(d / 4096)


def _ea_factor_np(port, d, n, steps, e, f, rho=0.95):
    """EA factor (kfactor.hpp:33-41, zero init) from the reference RNG's synthetic samples; the
    d x d x n products go through numpy's BLAS (input construction only -- ea_update parity is tested in
    test_gpu_parity.py)."""
    x = np.zeros((d, d))
    for k in range(steps):
        m = port.synthetic_m(ROOT_SEED, k, f, n, d, e)
        x = rho * x + (1.0 - rho) * (m @ m.T)
        x = 0.5 * (x + x.T)
    return x


# ---------------------------------------------------------------------------------------------- config 2
def test_config2_wide_pair_matches_oracle(port, cuda):
    import oracle
    import paper_2206_15397_b200 as rk

    d, n, e, steps, r, p, q, lam = 4096, 128, 0.8, 50, 220, 10, 4, 0.1
    xs = oracle.parallel_map(lambda f: _ea_factor_np(port, d, n, steps, e, f), [0, 1], 2)
    step = rk.BatchedStep([rk.LayerSpec(d, d)], rank=r, oversampling=p, power_iters=q,
                          method=rk.DecompMethod.SREVD, device=0)
    for f in (0, 1):
        step.factors[f].copy_(_t32(xs[f], cuda))
    j, _ = port.sample_gaussian(port.substream(GRAD_ROOT, 0, 0), 0, d, d)
    step.grads[0].copy_(_t32(j, cuda))
    step.decompose(OMEGA_ROOT, 0)
    step.precondition(lam)
    import torch

    torch.cuda.synchronize()
    decs = oracle.parallel_map(
        lambda f: port.srevd(xs[f], r, p, q, port.substream(OMEGA_ROOT, 0, f), 0), [0, 1], 2)
    for f in (0, 1):
        u0, d0, _ = decs[f]
        lr = step.lowrank(f)
        u1, d1 = _np64(lr.u), _np64(lr.d)
        assert recon_err(u1, d1, u0, d0) < TOL
        assert eig_err(d1, d0) < TOL
        assert orth_err(u1) < _orth_tol(d)
    s0 = port.precondition(decs[0][0], decs[0][1], decs[1][0], decs[1][1], lam, j)
    assert rel_fro(_np64(step.outs[0]), s0) < TOL


# ---------------------------------------------------------------------------------------------- config 4
VGG_A = [28, 577, 577, 1153, 1153, 2305, 2305, 2305, 4609, 4609, 4609, 4609, 4609, 513, 513, 513]
VGG_G = [64, 64, 128, 128, 256, 256, 256, 512, 512, 512, 512, 512, 512, 512, 512, 10]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_config4_sharded_step_is_bitwise_the_one_gpu_step(cuda, world):
    import torch

    import paper_2206_15397_b200 as rk
    from paper_2206_15397_b200.partition import GatherLayout, layer_cost, lpt_partition

    layers = list(zip(VGG_A, VGG_G))
    r, p, q, lam, n, warm = 220, 10, 4, 0.1, 128, 2
    kw = dict(rank=r, oversampling=p, power_iters=q, method=rk.DecompMethod.SREVD, n_samples=[n], device=0)
    g = torch.Generator(device="cuda").manual_seed(11)
    nf = 2 * len(layers)
    dims = [d for a, gd in layers for d in (a, gd)]
    # per-factor samples of every EA step and the gradients: the same tensors feed the 1-GPU and the shard plans
    samples = [[(torch.randn(d, n, device=cuda, generator=g) *
                 torch.arange(1, d + 1, device=cuda).pow(-1.0)[:, None] / math.sqrt(n)) for d in dims]
               for _ in range(warm)]
    grads = [torch.randn(gd, a, device=cuda, generator=g) for a, gd in layers]

    def run(layer_ids):
        specs = [rk.LayerSpec(*layers[l]) for l in layer_ids]
        tags = [2 * l + w for l in layer_ids for w in (0, 1)]
        st = rk.BatchedStep(specs, factor_indices=tags, **kw)
        for k in range(warm):
            for i, f in enumerate(tags):
                st.samples[i].copy_(samples[k][f])
            if k + 1 < warm:
                st.ea_update(0.95, 1.0)
        for i, l in enumerate(layer_ids):
            st.grads[i].copy_(grads[l])
        st.step(OMEGA_ROOT, 0, lam, 0.95, 1.0)
        torch.cuda.synchronize()
        out = {l: st.outs[i].clone() for i, l in enumerate(layer_ids)}
        bases = {f: (st.bases_t[i].clone(), st.dvals[i].clone()) for i, f in enumerate(tags)}
        del st
        return out, bases

    ref_out, ref_bases = run(list(range(len(layers))))
    parts = lpt_partition([layer_cost(a, gd, r, p) for a, gd in layers], world)
    sizes = [a * gd for a, gd in layers]
    layout = GatherLayout.build(sizes, parts)
    recv = torch.zeros(world * layout.chunk, device=cuda)
    for rank, mine in enumerate(parts):
        if not mine:
            continue
        out, bases = run(mine)
        send = recv[rank * layout.chunk:(rank + 1) * layout.chunk]  # the rank's slot of the all-gather
        for l in mine:
            send[layout.offsets[l]:layout.offsets[l] + sizes[l]].copy_(out[l].view(-1))
        for f, (bt, dv) in bases.items():
            assert torch.equal(bt, ref_bases[f][0]) and torch.equal(dv, ref_bases[f][1]), f"factor {f}"
    for l, (a, gd) in enumerate(layers):
        o = layout.owner[l]
        got = recv[o * layout.chunk + layout.offsets[l]:o * layout.chunk + layout.offsets[l] + sizes[l]]
        assert torch.equal(got.view(gd, a), ref_out[l]), f"layer {l}"


# ---------------------------------------------------------------------------------------------- config 5
def _srevd_fp64(x, omega, q, r):
    """rnla.hpp:47-56 + 90-105 restated in torch FP64 (Householder QR from cuSOLVER: any orthonormal basis of the
    same span gives the same U L U^T)."""
    import torch

    qb = torch.linalg.qr(x @ omega).Q
    for _ in range(q):
        z = torch.linalg.qr(x.T @ qb).Q
        qb = torch.linalg.qr(x @ z).Q
    c = qb.T @ (x @ qb)
    c = 0.5 * (c + c.T)
    lam, pm = torch.linalg.eigh(c)
    lam, pm = lam.flip(0)[:r], pm.flip(1)[:, :r]
    return qb @ pm, lam.clamp_min(0.0)


def _apply_fp64(u, dv, lam, v, left):
    """kfactor.hpp:134-161 (Eq. 11) in FP64."""
    b = 1.0 / (dv + lam) - 1.0 / lam
    if left:
        return u @ (b[:, None] * (u.T @ v)) + v / lam
    return ((v @ u) * b[None, :]) @ u.T + v / lam


def test_config5_very_wide_pair_matches_fp64_restatement(port, cuda):
    import torch

    import paper_2206_15397_b200 as rk

    d, n, e, steps, r, p, q, lam = 16384, 512, 1.2, 10, 256, 16, 4, 0.05
    w = r + p
    s = torch.arange(1, d + 1, device=cuda, dtype=torch.float64).pow(-e)
    step = rk.BatchedStep([rk.LayerSpec(d, d)], rank=r, oversampling=p, power_iters=q,
                          method=rk.DecompMethod.SREVD, device=0)
    xs64 = []
    for f in (0, 1):
        x = torch.zeros(d, d, device=cuda, dtype=torch.float64)
        for k in range(steps):
            z = torch.randn(n, d, device=cuda, dtype=torch.float64,
                            generator=torch.Generator(device="cuda").manual_seed(1000 * f + k))
            m = (z * s[None, :]).T / math.sqrt(n)
            x = 0.95 * x + 0.05 * (m @ m.T)
            x = 0.5 * (x + x.T)
        step.factors[f].copy_(x.float())
        xs64.append(x.float().double())  # the GPU path sees the FP32 factor: restate on exactly that input
        del x
    j = torch.randn(d, d, device=cuda, generator=torch.Generator(device="cuda").manual_seed(5))
    step.grads[0].copy_(j)
    step.decompose(OMEGA_ROOT, 0)
    step.precondition(lam)
    torch.cuda.synchronize()
    ref = []
    for f in (0, 1):
        om, _ = port.sample_gaussian(port.substream(OMEGA_ROOT, 0, f), 0, d, w)  # rng.hpp Omega, FP64
        u0, d0 = _srevd_fp64(xs64[f], torch.as_tensor(om, device=cuda), q, r)
        ref.append((u0, d0))
        lr = step.lowrank(f)
        u1, d1 = lr.u.double(), lr.d.double()
        rec1, rec0 = (u1 * d1[None, :]) @ u1.T, (u0 * d0[None, :]) @ u0.T
        assert float(torch.linalg.norm(rec1 - rec0) / torch.linalg.norm(rec0)) < TOL
        assert float(((d1 - d0).abs() / d0.abs()).max()) < TOL
        assert float((u1.T @ u1 - torch.eye(r, device=cuda, dtype=torch.float64)).abs().max()) < _orth_tol(d)
        del rec1, rec0
    (ua, da), (ug, dg) = ref
    s0 = _apply_fp64(ug, dg, lam, _apply_fp64(ua, da, lam, j.double(), left=False), left=True)
    s1 = step.outs[0].double()
    assert float(torch.linalg.norm(s1 - s0) / torch.linalg.norm(s0)) < TOL


def test_config5_size_exact_low_rank_recovery_and_eq11_identity(cuda):
    """Size-independent properties at d = 16384: an exactly rank-200 factor (< r = 256) is recovered to FP32
    accuracy, and the damped inverse maps each recovered eigenvector u_i to u_i / (d_i + lam)."""
    import torch

    import paper_2206_15397_b200 as rk

    d, k, r, p, q, lam = 16384, 200, 256, 16, 4, 0.05
    g = torch.Generator(device="cuda").manual_seed(21)
    v = torch.linalg.qr(torch.randn(d, k, device=cuda, dtype=torch.float64, generator=g)).Q
    ev = 0.8 ** torch.arange(k, device=cuda, dtype=torch.float64) + 1e-3
    x = ((v * ev[None, :]) @ v.T).float()
    lr = rk.srevd(x, rk.SketchParams(r, p, q), rk.RngState(rk.substream_seed(OMEGA_ROOT, 0, 0)))
    torch.cuda.synchronize()
    u, dv = lr.u.double(), lr.d.double()
    xr = (u * dv[None, :]) @ u.T
    # 3xTF32 with FP32 accumulation (slices of <= 1024 K): measured 4.9e-5 at d = 16384 (FP64 restatement 2.5e-8)
    assert float(torch.linalg.norm(xr - x.double()) / torch.linalg.norm(x.double())) < TOL
    assert float(((dv[:k] - ev).abs() / ev).max()) < 1e-4
    assert float(dv[k:].abs().max()) < 1e-5 * float(ev[0])
    top = lr.u[:, :16].contiguous()
    out = rk.apply_lowrank_damped_inverse(lr, lam, top, rk.ApplySide.LEFT)
    expect = top.double() / (dv[:16][None, :] + lam)
    assert float(torch.linalg.norm(out.double() - expect) / torch.linalg.norm(expect)) < TOL  # measured 1.4e-5


def test_cta_pair_kernel_is_bitwise_the_single_cta_kernels_on_unaligned_shapes():
    """The X*Q products on CTA pairs (tcgen05 cta_group::2) keep every element's K order: a step over 32 factors whose
    dimensions sit off every tile boundary hashes identically with RKFAC_XQ_PAIR=1 and =0 (the switch is read once per
    process, hence the two subprocesses; tools/pair_bitwise.py)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for pair in ("1", "0"):
        env = dict(os.environ, RKFAC_XQ_PAIR=pair)
        res = subprocess.run([sys.executable, os.path.join(root, "tools", "pair_bitwise.py"), "2", "1", "mixed"],
                             env=env, capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        outs.append(res.stdout.strip().splitlines())
    assert len(outs[0]) == 2 and outs[0] == outs[1]
