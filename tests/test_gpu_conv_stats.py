"""Convolution factor statistics feeding the batched EA: the GPU producer (csrc/stats.cu) against a
numpy im2col restatement, and the plan's long-n EA (n = B*H*W > 512: K slices of 512 + the reference's symmetrize,
kfactor.hpp:33-41) against the oracle's ea_update, then the whole step (rand-EVD + preconditioning) against the
oracle on the conv layers' factors.

Conventions restated from network.hpp: A = [patches; 1] (with_ones_row, :94-95), G = output gradient (:134), each
scaled by 1/sqrt(n) before ea_update (accumulate_factors, :155-165), n = B*Ho*Wo output locations (KFC)."""
import math

import numpy as np
import pytest

from tests.helpers import GRAD_ROOT, OMEGA_ROOT, eig_err, recon_err, rel_fro

pytestmark = pytest.mark.gpu

EA_TOL = 3e-8 * 512  # K slices of 512 (tests/test_gpu_ea_step.py: 3e-8 per unit of accumulation length)


def im2col_ref(x, kh, kw, stride, pad):
    """numpy restatement: rows (c, ky, kx), columns (b, oy, ox), plus the ones row (network.hpp:94-95)."""
    B, C, H, W = x.shape
    Ho = (H + 2 * pad - kh) // stride + 1
    Wo = (W + 2 * pad - kw) // stride + 1
    xp = np.zeros((B, C, H + 2 * pad, W + 2 * pad), x.dtype)
    xp[:, :, pad:pad + H, pad:pad + W] = x
    out = np.empty((C * kh * kw + 1, B * Ho * Wo), x.dtype)
    for c in range(C):
        for ky in range(kh):
            for kx in range(kw):
                patch = xp[:, c, ky:ky + stride * Ho:stride, kx:kx + stride * Wo:stride]  # B x Ho x Wo
                out[(c * kh + ky) * kw + kx] = patch.reshape(-1)
    out[-1] = 1.0
    return out


LAYERS = [  # (B, Cin, H, W, Cout, k, stride, pad): a VGG-like first conv and a deeper one, n > 512 both
    (4, 3, 32, 32, 64, 3, 1, 1),
    (8, 16, 12, 12, 32, 3, 1, 1),
    (8, 24, 8, 8, 40, 3, 2, 1),
]


def _inputs(port, k, l, B, Cin, H, W, Cout, kk, st, pd):
    x, _ = port.sample_gaussian(port.substream(31, k, 2 * l), 0, B * Cin, H * W)
    Ho = (H + 2 * pd - kk) // st + 1
    Wo = (W + 2 * pd - kk) // st + 1
    dy, _ = port.sample_gaussian(port.substream(31, k, 2 * l + 1), 0, B * Cout, Ho * Wo)
    return (np.maximum(x, 0.0).reshape(B, Cin, H, W).astype(np.float32),
            dy.reshape(B, Cout, Ho, Wo).astype(np.float32), Ho, Wo)


def test_conv_patches_are_bitwise_the_im2col_restatement(port, cuda):
    import torch
    from paper_2206_15397_b200.kfac import conv_factor_statistics

    for l, (B, Cin, H, W, Cout, kk, st, pd) in enumerate(LAYERS):
        x, dy, Ho, Wo = _inputs(port, 0, l, B, Cin, H, W, Cout, kk, st, pd)
        a, g = conv_factor_statistics(torch.as_tensor(x, device=cuda), torch.as_tensor(dy, device=cuda), kk, st, pd)
        torch.cuda.synchronize()
        n = B * Ho * Wo
        sc = np.float32(1.0 / math.sqrt(n))
        a_ref = im2col_ref(x, kk, kk, st, pd) * sc
        g_ref = dy.transpose(1, 0, 2, 3).reshape(Cout, n) * sc
        assert np.array_equal(a.cpu().numpy(), a_ref), l
        assert np.array_equal(g.cpu().numpy(), g_ref), l


def test_conv_statistics_through_the_plan_match_the_oracle(port, cuda):
    """3 EA steps from zero on the conv statistics (long n: sliced + symmetrised), then srevd of every factor and the
    RIGHT_A / LEFT_G preconditioning of every layer, vs the oracle on the same FP32-valued statistics."""
    import torch
    import paper_2206_15397_b200 as rk
    from paper_2206_15397_b200.kfac import conv_factor_statistics, conv_output_size

    specs, ns = [], []
    for (B, Cin, H, W, Cout, kk, st, pd) in LAYERS:
        Ho, Wo = conv_output_size(H, W, kk, st, pd)
        specs.append(rk.LayerSpec(Cin * kk * kk + 1, Cout))
        ns += [B * Ho * Wo] * 2
    r, p, q, lam = 24, 6, 2, 0.1
    step = rk.BatchedStep(specs, rank=r, oversampling=p, power_iters=q, method=rk.DecompMethod.SREVD,
                          n_samples=ns, device=0)
    xs = [np.zeros((d, d)) for d in step.dims]
    for k in range(3):
        ms = []
        for l, (B, Cin, H, W, Cout, kk, st, pd) in enumerate(LAYERS):
            x, dy, _, _ = _inputs(port, k, l, B, Cin, H, W, Cout, kk, st, pd)
            conv_factor_statistics(torch.as_tensor(x, device=cuda), torch.as_tensor(dy, device=cuda), kk, st, pd,
                                   out_a=step.samples[2 * l], out_g=step.samples[2 * l + 1])
            ms += [step.samples[2 * l].double().cpu().numpy(), step.samples[2 * l + 1].double().cpu().numpy()]
        step.ea_update(0.95, 1.0)
        xs = [port.ea_update(xs[f], ms[f], 0.95) for f in range(len(xs))]
    torch.cuda.synchronize()
    for f in range(len(xs)):
        got = step.factors[f].double().cpu().numpy()
        assert np.array_equal(got, got.T), f  # symmetrize_in_place: exact
        assert rel_fro(got, xs[f]) < EA_TOL, (f, rel_fro(got, xs[f]))
    grads = []
    for l, L in enumerate(specs):
        j, _ = port.sample_gaussian(port.substream(GRAD_ROOT, l, 0), 0, L.dim_g, L.dim_a)
        grads.append(j)
        step.grads[l].copy_(torch.as_tensor(j, dtype=torch.float32, device=cuda))
    step.decompose(OMEGA_ROOT, 0)
    step.precondition(lam)
    torch.cuda.synchronize()
    xg = [step.factors[f].double().cpu().numpy() for f in range(len(xs))]  # same inputs on both sides
    for l in range(len(specs)):
        decs = []
        for w in (0, 1):
            f = 2 * l + w
            u0, d0, _ = port.srevd(xg[f], r, p, q, port.substream(OMEGA_ROOT, 0, f), 0)
            lr = step.lowrank(f)
            assert recon_err(lr.u.double().cpu().numpy(), lr.d.double().cpu().numpy(), u0, d0) < 1e-4
            assert eig_err(lr.d.double().cpu().numpy(), d0) < 1e-4
            decs.append((u0, d0))
        s0 = port.precondition(decs[0][0], decs[0][1], decs[1][0], decs[1][1], lam, grads[l])
        assert rel_fro(step.outs[l].double().cpu().numpy(), s0) < 1e-4
