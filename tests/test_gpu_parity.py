"""GPU parity: the CUDA path through the C-ABI vs the CPU oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): preconditioned gradient rel. Frobenius <= 1e-4 in FP32 (our GEMMs accumulate
in FP32; the first orthonormalisations and the eigensolver run in FP64), the same bar for the sign-invariant
reconstruction U L U^T and the top-r eigenvalues (max relative error) on zero-init factors.
"""
import numpy as np
import pytest

from tests.helpers import (GRAD_ROOT, OMEGA_ROOT, build_factor, eig_err, geometric_spectrum, orth_err,
                           psd_with_spectrum, recon_err, rel_fro)

pytestmark = pytest.mark.gpu

TOL = 1e-4


def t32(a, dev):
    import torch

    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32), device=dev)


def np64(t):
    return t.detach().double().cpu().numpy()


# ------------------------------------------------------------------------------------------------ Omega
def test_sample_gaussian_matches_reference_stream(port, cuda):
    import paper_2206_15397_b200 as rk

    seed = port.substream(OMEGA_ROOT, 0, 0)
    rng = rk.RngState(seed, 0)
    g = rk.sample_gaussian(rng, 300, 74, device=cuda)
    assert rng.counter == 2 * 300 * 74
    ref, ctr = port.sample_gaussian(seed, 0, 300, 74)
    assert ctr == rng.counter
    got = np64(g)
    # FP64 math on both sides, FP32 store: identical except (rarely) one FP32 ulp at a rounding boundary.
    ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(got - ref.astype(np.float32).astype(np.float64)) <= ulp)
    assert np.mean(got == ref.astype(np.float32)) > 0.999
    # known answers: Omega[0][0..3], Omega[1][0] for RngState(7).substream(0,0), w=74
    assert got[0, :4] == pytest.approx([-0.061239146505972855, -0.41276414698843211, 1.1755512626931139,
                                        -1.1985571924273768], rel=1e-6)
    assert got[1, 0] == pytest.approx(1.2097400634173616, rel=1e-6)


# --------------------------------------------------------------------------------------------------- EA
def test_ea_update_matches_oracle(port, cuda):
    import paper_2206_15397_b200 as rk

    d, n = 333, 96
    f = rk.EAKFactor.create(d, 0.95, zero_init=False, device=cuda)
    x = np.eye(d)
    for k in range(5):
        m = port.synthetic_m(11, k, 0, n, d, 0.7)
        rk.ea_update(f, t32(m, cuda))
        x = port.ea_update(x, m, 0.95)
    got = np64(f.mbar)
    assert rel_fro(got, x) < 1e-6
    assert np.array_equal(got, got.T)  # exactly symmetric (kfactor.hpp:39)
    assert f.steps == 5


def test_ea_update_zero_and_no_memory_cases(port, cuda):
    """test_kfactor.cpp:17-29."""
    import torch
    import paper_2206_15397_b200 as rk

    f = rk.EAKFactor.create(3, 0.95, device=cuda)
    rk.ea_update(f, torch.zeros(3, 2, device=cuda))
    assert np.abs(np64(f.mbar) - 0.95 * np.eye(3)).max() <= 1e-7
    m, _ = port.sample_gaussian(1, 0, 3, 2)
    g = rk.EAKFactor.create(3, 0.0, device=cuda)
    rk.ea_update(g, t32(m, cuda))
    # 3xTF32 on the tensor cores: relative to the entries (|m m^T| ~ 5 here), ~2^-21 per product
    assert np.abs(np64(g.mbar) - m @ m.T).max() <= 1e-6 * max(1.0, np.abs(m @ m.T).max())


def test_ea_update_dimension_check(cuda):
    """test_kfactor.cpp:31-34."""
    import torch
    import paper_2206_15397_b200 as rk

    f = rk.EAKFactor.create(3, 0.9, device=cuda)
    with pytest.raises(rk.DimensionMismatch):
        rk.ea_update(f, torch.zeros(4, 2, device=cuda))


# ------------------------------------------------------------------------------------ decompositions
@pytest.fixture(scope="module")
def config1(port):
    """BASELINE config 1: d=512, 20 EA steps of X^T X / 256, s_i = i^-1, zero init."""
    return build_factor(port, 512, 256, 20, 1.0)


@pytest.mark.parametrize("method", ["srevd", "rsvd_psd"])
def test_decomposition_config1_parity(port, cuda, config1, method):
    import paper_2206_15397_b200 as rk

    x = config1
    seed = port.substream(OMEGA_ROOT, 0, 0)
    u0, d0, c0 = getattr(port, method)(x, 64, 10, 2, seed, 0)
    rng = rk.RngState(seed, 0)
    lr = getattr(rk, method)(t32(x, cuda), rk.SketchParams(64, 10, 2), rng)
    assert rng.counter == c0
    u1, d1 = np64(lr.u), np64(lr.d)
    assert u1.shape == u0.shape
    e_rec = recon_err(u1, d1, u0, d0)
    e_eig = eig_err(d1, d0)
    assert e_rec < TOL, e_rec
    assert e_eig < TOL, e_eig
    # rsvd_psd's basis is Y P / s (eig.hpp:260-266): FP32 rounding of Y is amplified by s_1/s_r (~4e3 here)
    assert orth_err(u1) < (1e-5 if method == "srevd" else 1e-4)
    assert np.all(np.diff(d1) <= 1e-6 * d1[0])  # descending


def test_precondition_config1_parity(port, cuda, config1):
    import paper_2206_15397_b200 as rk

    x = config1
    seed = port.substream(OMEGA_ROOT, 0, 0)
    u0, d0, _ = port.srevd(x, 64, 10, 2, seed, 0)
    j, _ = port.sample_gaussian(port.substream(GRAD_ROOT, 0, 0), 0, 512, 512)
    s0 = port.precondition(u0, d0, u0, d0, 0.1, j)
    lr = rk.srevd(t32(x, cuda), rk.SketchParams(64, 10, 2), rk.RngState(seed, 0))
    mid = rk.apply_lowrank_damped_inverse(lr, 0.1, t32(j, cuda), rk.ApplySide.RIGHT)
    s1 = rk.apply_lowrank_damped_inverse(lr, 0.1, mid, rk.ApplySide.LEFT)
    assert rel_fro(np64(s1), s0) < TOL


# ----------------------------------------------------------------------- reference unit-test behaviour
def test_srevd_exact_low_rank_and_isotropic(cuda):
    """test_rnla.cpp:53-70."""
    import paper_2206_15397_b200 as rk

    x = np.diag([5.0, 4.0, 0.0, 0.0])
    lr = rk.srevd(t32(x, cuda), rk.SketchParams(2, 1, 1), rk.RngState(3))
    d = np64(lr.d); u = np64(lr.u)
    assert d[0] == pytest.approx(5.0, abs=1e-5) and d[1] == pytest.approx(4.0, abs=1e-5)
    assert np.abs(u[2:, :]).max() <= 1e-5
    iso = rk.srevd(t32(np.eye(4), cuda), rk.SketchParams(2, 1, 0), rk.RngState(3))
    assert np64(iso.d) == pytest.approx([1.0, 1.0], abs=1e-5)


def test_rsvd_psd_rank1(port, cuda):
    """test_rnla.cpp:72-88."""
    import paper_2206_15397_b200 as rk

    v, _ = port.sample_gaussian(21, 0, 6, 1)
    v = v * (2.0 / np.linalg.norm(v))
    x = v @ v.T
    lr = rk.rsvd_psd(t32(x, cuda), rk.SketchParams(1, 1, 1), rk.RngState(5))
    assert np64(lr.d)[0] == pytest.approx(4.0, abs=1e-5)
    u = np64(lr.u)[:, 0]
    sign = 1.0 if u[0] * v[0, 0] > 0 else -1.0
    assert np.abs(u * sign - v[:, 0] / 2.0).max() <= 1e-5


def test_exact_recovery_when_rank_below_r(port, cuda):
    """test_rnla.cpp:142-153 (rank-5 X, sketch 5+3: rank-deficient orthonormalisation)."""
    import paper_2206_15397_b200 as rk

    g, _ = port.sample_gaussian(31, 0, 30, 5)
    x = g @ g.T
    x = 0.5 * (x + x.T)
    nx = np.linalg.norm(x)
    for seed in range(4):
        for fn in (rk.rsvd_psd, rk.srevd):
            lr = fn(t32(x, cuda), rk.SketchParams(5, 3, 1), rk.RngState(seed))
            u, d = np64(lr.u), np64(lr.d)
            assert np.linalg.norm(x - (u * d) @ u.T) <= 1e-5 * nx


def test_sketch_clamping(cuda):
    """test_rnla.cpp:155-162."""
    import paper_2206_15397_b200 as rk

    x = np.diag([4.0, 3.0, 2.0, 1.0])
    lr = rk.rsvd_psd(t32(x, cuda), rk.SketchParams(10, 10, 1), rk.RngState(17))
    assert lr.rank() == 4
    u, d = np64(lr.u), np64(lr.d)
    assert np.abs(x - (u * d) @ u.T).max() <= 1e-5


def test_orthonormality_and_ordering(port, cuda):
    """test_rnla.cpp:130-140."""
    import paper_2206_15397_b200 as rk

    x = psd_with_spectrum(port, geometric_spectrum(40), 7)
    a = rk.rsvd_psd(t32(x, cuda), rk.SketchParams(8, 4, 2), rk.RngState(1))
    b = rk.srevd(t32(x, cuda), rk.SketchParams(8, 4, 2), rk.RngState(1))
    assert orth_err(np64(a.u)) <= 1e-5
    assert orth_err(np64(b.u)) <= 1e-5
    da = np64(a.d)
    assert np.all(da[1:] <= da[:-1] + 1e-7)
    assert np64(b.d)[-1] >= 0.0


def test_determinism(port, cuda):
    """test_rnla.cpp:164-172: same inputs and seed reproduce outputs bit for bit."""
    import paper_2206_15397_b200 as rk

    x = t32(psd_with_spectrum(port, geometric_spectrum(30), 2), cuda)
    a = rk.rsvd_psd(x, rk.SketchParams(6, 4, 2), rk.RngState(6))
    b = rk.rsvd_psd(x, rk.SketchParams(6, 4, 2), rk.RngState(6))
    assert np.array_equal(np64(a.u), np64(b.u)) and np.array_equal(np64(a.d), np64(b.d))


def test_geometric_spectrum_matches_oracle(port, cuda):
    """test_rnla.cpp:40-51 setting (100x100, r=10, p=10, q=4), GPU vs oracle with the same Omega."""
    import paper_2206_15397_b200 as rk

    x = psd_with_spectrum(port, geometric_spectrum(100), 123)
    for seed in range(3):
        for name in ("rsvd_psd", "srevd"):
            u0, d0, _ = getattr(port, name)(x, 10, 10, 4, seed, 0)
            lr = getattr(rk, name)(t32(x, cuda), rk.SketchParams(10, 10, 4), rk.RngState(seed))
            assert recon_err(np64(lr.u), np64(lr.d), u0, d0) < TOL
            assert eig_err(np64(lr.d), d0) < TOL


# ------------------------------------------------------------------------------------------------ apply
def test_apply_diagonal_special_cases(cuda):
    """test_kfactor.cpp:142-158."""
    import torch
    import paper_2206_15397_b200 as rk

    lam = 0.25
    full = rk.LowRankEig(torch.eye(3, device=cuda), torch.tensor([3.0, 2.0, 1.0], device=cuda))
    v = torch.arange(1, 7, dtype=torch.float32, device=cuda).reshape(3, 2)
    out = np64(rk.apply_lowrank_damped_inverse(full, lam, v, rk.ApplySide.LEFT))
    expect = np64(v) / (np.array([3.0, 2.0, 1.0])[:, None] + lam)
    # Eq. 11 forms V/lam + U b U^T V: FP32 (3xTF32) rounding relative to the terms' size, |V|/lam = 24 here
    bar = 1e-6 * max(1.0, np.abs(np64(v)).max() / lam)
    assert np.abs(out - expect).max() <= bar
    zero = rk.LowRankEig(torch.eye(3, device=cuda)[:, :2].contiguous(), torch.zeros(2, device=cuda))
    out2 = np64(rk.apply_lowrank_damped_inverse(zero, lam, v, rk.ApplySide.LEFT))
    assert np.abs(out2 - np64(v) / lam).max() <= bar


@pytest.mark.parametrize("lam", [1e-3, 1e-1, 1.0, 10.0])
def test_apply_matches_oracle(port, cuda, lam):
    """test_kfactor.cpp:160-177 shapes, GPU vs oracle (FP64)."""
    import paper_2206_15397_b200 as rk

    for seed in range(3):
        g, _ = port.sample_gaussian(seed, 0, 20, 5)
        q, _ = port.qr_thin(g)
        d = np.array([2.0, 1.5, 1.0, 0.5, 0.25])
        v, _ = port.sample_gaussian(seed, 200, 20, 7)
        ref = port.apply_lowrank_damped_inverse(q, d, lam, v, "left")
        lr = rk.LowRankEig(t32(q, cuda), t32(d[None, :], cuda)[0])
        got = np64(rk.apply_lowrank_damped_inverse(lr, lam, t32(v, cuda), rk.ApplySide.LEFT))
        assert rel_fro(got, ref) < 1e-5


def test_apply_left_right_duality(port, cuda):
    """test_kfactor.cpp:179-190."""
    import paper_2206_15397_b200 as rk

    g, _ = port.sample_gaussian(8, 0, 12, 4)
    q, _ = port.qr_thin(g)
    lr = rk.LowRankEig(t32(q, cuda), t32(np.array([[3.0, 2.0, 1.0, 0.5]]), cuda)[0])
    v, _ = port.sample_gaussian(8, 100, 5, 12)
    right = np64(rk.apply_lowrank_damped_inverse(lr, 0.3, t32(v, cuda), rk.ApplySide.RIGHT))
    left_t = np64(rk.apply_lowrank_damped_inverse(lr, 0.3, t32(v.T, cuda), rk.ApplySide.LEFT)).T
    assert np.abs(right - left_t).max() <= 1e-6 * np.abs(right).max()


def test_damping_must_be_positive(cuda):
    """test_kfactor.cpp:192-199."""
    import torch
    import paper_2206_15397_b200 as rk

    lr = rk.LowRankEig(torch.eye(2, device=cuda), torch.ones(2, device=cuda))
    v = torch.ones(2, 1, device=cuda)
    for lam in (0.0, -1.0):
        with pytest.raises(rk.DampingNonpositive):
            rk.apply_lowrank_damped_inverse(lr, lam, v, rk.ApplySide.LEFT)


# ------------------------------------------------------------------------------------ batched plan
def test_batched_step_matches_per_layer_oracle(port, cuda):
    """All factors of all layers in single launches == the reference's per-layer loop (optimizer.hpp:139-167)."""
    import torch
    import paper_2206_15397_b200 as rk

    layers = [rk.LayerSpec(28, 64), rk.LayerSpec(577, 64), rk.LayerSpec(513, 10), rk.LayerSpec(300, 257)]
    r, p, q, lam, n = 40, 10, 2, 0.1, 64
    step = rk.BatchedStep(layers, rank=r, oversampling=p, power_iters=q, method=rk.DecompMethod.SREVD,
                          n_samples=[n], device=0)
    xs = []
    for f, d in enumerate(step.dims):
        x = build_factor(port, d, n, 3, 1.0, f=f)
        xs.append(x)
        step.factors[f].copy_(t32(x, cuda))
    grads = []
    for l, L in enumerate(layers):
        j, _ = port.sample_gaussian(port.substream(GRAD_ROOT, l, 0), 0, L.dim_g, L.dim_a)
        grads.append(j)
        step.grads[l].copy_(t32(j, cuda))
    step.decompose(OMEGA_ROOT, 0)
    step.precondition(lam)
    torch.cuda.synchronize()
    for l, L in enumerate(layers):
        decs = []
        for which in (0, 1):
            f = 2 * l + which
            seed = port.substream(OMEGA_ROOT, 0, f)
            u0, d0, _ = port.srevd(xs[f], r, p, q, seed, 0)
            lr = step.lowrank(f)
            assert recon_err(np64(lr.u), np64(lr.d), u0, d0) < TOL
            assert eig_err(np64(lr.d), d0) < TOL
            decs.append((u0, d0))
        s0 = port.precondition(decs[0][0], decs[0][1], decs[1][0], decs[1][1], lam, grads[l])
        assert rel_fro(np64(step.outs[l]), s0) < TOL


@pytest.mark.parametrize("d,e,steps", [(1153, 0.0, 6), (1153, 1.0, 20)])
def test_batched_step_large_factor_vgg_sketch(port, cuda, d, e, steps):
    """VGG16 sketch sizes (r=220, p=10, q=4) on a factor large enough for split-K Gram products, for an isotropic
    (e=0: well conditioned, slowly decaying) and a decaying (e=1) spectrum."""
    import torch
    import paper_2206_15397_b200 as rk

    r, p, q, n = 220, 10, 4, 128
    step = rk.BatchedStep([rk.LayerSpec(d, 64)], rank=r, oversampling=p, power_iters=q,
                          method=rk.DecompMethod.SREVD, n_samples=[n], device=0)
    x = build_factor(port, d, n, steps, e, f=0)
    step.factors[0].copy_(t32(x, cuda))
    step.factors[1].copy_(t32(build_factor(port, 64, n, steps, e, f=1), cuda))
    step.decompose(OMEGA_ROOT, 0)
    torch.cuda.synchronize()
    u0, d0, _ = port.srevd(x, r, p, q, port.substream(OMEGA_ROOT, 0, 0), 0)
    lr = step.lowrank(0)
    assert recon_err(np64(lr.u), np64(lr.d), u0, d0) < TOL
    assert eig_err(np64(lr.d), d0) < TOL
    assert orth_err(np64(lr.u)) < 1e-5


def test_rank_deficient_ea_start_is_fast_and_exact(port, cuda):
    """First K-FAC step from zero-init EA: rank(X) = n = 128 < w = 230, so ~100 sketch columns are
    rank deficient in every orthonormalisation.  The decomposition must stay exact on range(X) (recovery of X to
    FP32 accuracy) and must not fall off a performance cliff (the completion runs once, on the final basis)."""
    import time

    import torch
    import paper_2206_15397_b200 as rk

    d, n, r, p, q = 1153, 128, 220, 10, 4
    step = rk.BatchedStep([rk.LayerSpec(d, 64)], rank=r, oversampling=p, power_iters=q,
                          method=rk.DecompMethod.SREVD, n_samples=[n], device=0)
    x = build_factor(port, d, n, 1, 1.0, f=0)  # one EA update from zero: rank 128
    step.factors[0].copy_(t32(x, cuda))
    step.factors[1].copy_(t32(build_factor(port, 64, n, 1, 1.0, f=1), cuda))
    step.decompose(OMEGA_ROOT, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step.decompose(OMEGA_ROOT, 0)
    torch.cuda.synchronize()
    elapsed = time.perf_counter() - t0
    lr = step.lowrank(0)
    u, dv = np64(lr.u), np64(lr.d)
    assert np.linalg.norm(x - (u * dv) @ u.T) <= 1e-5 * np.linalg.norm(x)
    # the ~100 null-space columns are eigenvectors of FP32-noise-level eigenvalues of the core: orthonormal to a few
    # FP32 ulps times sqrt(w) rather than to one
    assert orth_err(u) < 5e-5
    assert elapsed < 0.1, elapsed


def test_streamed_step_is_bitwise_the_batched_step(cuda):
    """Layer groups on separate streams (StreamedStep) give bitwise the single-plan result."""
    import math

    import torch
    import paper_2206_15397_b200 as rk

    layers = [rk.LayerSpec(577, 64), rk.LayerSpec(300, 257), rk.LayerSpec(28, 64), rk.LayerSpec(513, 10)]
    kw = dict(rank=40, oversampling=10, power_iters=2, method=rk.DecompMethod.SREVD, n_samples=[64], device=0)
    one = rk.BatchedStep(layers, **kw)
    two = rk.StreamedStep(layers, groups=2, **kw)
    g = torch.Generator(device="cuda").manual_seed(3)
    for f, d in enumerate(one.dims):
        s = torch.arange(1, d + 1, device=cuda, dtype=torch.float32).pow(-1.0)
        m = torch.randn(d, 64, device=cuda, generator=g) * s[:, None] / math.sqrt(64)
        one.samples[f].copy_(m)
        two.samples[f].copy_(m)
    for l, L in enumerate(layers):
        j = torch.randn(L.dim_g, L.dim_a, device=cuda, generator=g)
        one.grads[l].copy_(j)
        two.grads[l].copy_(j)
    for k in range(3):
        one.step(7, k, 0.1)
        two.step(7, k, 0.1)
    torch.cuda.synchronize()
    for f in range(len(one.dims)):
        assert torch.equal(one.factors[f], two.factors[f])
        assert torch.equal(one.bases_t[f], two.bases_t[f]) and torch.equal(one.dvals[f], two.dvals[f])
    for l in range(len(layers)):
        assert torch.equal(one.outs[l], two.outs[l])


def test_streamed_step_from_host_buffers_is_bitwise_the_step(cuda):
    """StreamedStep.step_host (pinned host inputs/outputs, gradients uploaded during the decomposition) == step()."""
    import math

    import torch
    import paper_2206_15397_b200 as rk

    layers = [rk.LayerSpec(577, 64), rk.LayerSpec(300, 257), rk.LayerSpec(28, 64)]
    kw = dict(rank=40, oversampling=10, power_iters=2, method=rk.DecompMethod.SREVD, n_samples=[64], device=0)
    st = rk.StreamedStep(layers, groups=2, **kw)
    g = torch.Generator(device="cuda").manual_seed(5)
    h_samples, h_grads = [], []
    for f, d in enumerate(st.dims):
        s = torch.arange(1, d + 1, device=cuda, dtype=torch.float32).pow(-1.0)
        h_samples.append((torch.randn(d, 64, device=cuda, generator=g) * s[:, None] / math.sqrt(64)).cpu().pin_memory())
    for L in layers:
        h_grads.append(torch.randn(L.dim_g, L.dim_a, device=cuda, generator=g).cpu().pin_memory())
    h_outs = [torch.empty(L.dim_g, L.dim_a).pin_memory() for L in layers]
    x0 = [x.clone() for x in st.factors]
    st.step_host(7, 0, 0.1, h_samples, h_grads, h_outs)
    torch.cuda.synchronize()
    got = [o.clone() for o in h_outs]
    for x, y in zip(st.factors, x0):
        x.copy_(y)
    for f in range(len(st.dims)):
        st.samples[f].copy_(h_samples[f])
    for l in range(len(layers)):
        st.grads[l].copy_(h_grads[l])
    st.step(7, 0, 0.1)
    torch.cuda.synchronize()
    for l in range(len(layers)):
        assert torch.equal(got[l], st.outs[l].cpu())


# ------------------------------------------------------------------------------------ exact K-FAC comparator
@pytest.mark.parametrize("side", ["left", "right"])
def test_exact_kfac_comparator_matches_oracle(port, cuda, side):
    """full eigendecomposition + apply_eig_damped_inverse (kfactor.hpp:165-186) vs the oracle's
    sym_eig (eig.hpp:210-237) and apply_eig_damped_inverse on the same EA factor."""
    import paper_2206_15397_b200 as rk

    d, lam = 384, 0.1
    x = build_factor(port, d, 128, 6, 1.0, f=0)
    p0, d0 = port.sym_eig(x)
    v, _ = port.sample_gaussian(port.substream(GRAD_ROOT, 0, 0), 0, d, 200) if side == "left" else \
        port.sample_gaussian(port.substream(GRAD_ROOT, 0, 0), 0, 200, d)
    s0 = port.apply_eig_damped_inverse(p0, d0, lam, v, side)
    eig = rk.sym_eig(t32(x, cuda))
    assert eig_err(np64(eig.d)[:50], d0[:50]) < TOL  # the well-resolved top of the spectrum
    s1 = rk.apply_eig_damped_inverse(eig, lam, t32(v, cuda), rk.ApplySide.LEFT if side == "left" else
                                     rk.ApplySide.RIGHT)
    assert rel_fro(np64(s1), s0) < TOL
    with pytest.raises(rk.DampingNonpositive):
        rk.apply_eig_damped_inverse(eig, 0.0, t32(v, cuda), rk.ApplySide.LEFT)


# ------------------------------------------------------------------------------- optimizer orchestration
@pytest.mark.parametrize("method", ["sre", "rs", "kfac"])
def test_kfac_optimizer_cache_and_schedule_match_oracle(port, cuda, method):
    """kfac.KfacOptimizer (identity-init EA through the plan, decomposition cache on T_KI) == the reference's
    optimizer loop restated with the oracle (optimizer.hpp:139-167, network.hpp:155-165)."""
    import math

    import torch
    import paper_2206_15397_b200 as rk
    from paper_2206_15397_b200.kfac import KfacOptimizer, Method, OptimizerConfig, ScheduleOverrides

    layers = [rk.LayerSpec(65, 48), rk.LayerSpec(49, 10)]
    n, r, p, q, lam, seed = 32, 24, 6, 2, 0.1, 11
    meth = {"sre": Method.SRE_KFAC, "rs": Method.RS_KFAC, "kfac": Method.KFAC}[method]
    cfg = OptimizerConfig(method=meth, n_pwr_it=q,
                          overrides=ScheduleOverrides(lam=lam, target_rank=r, oversampling=p, t_ki=10))
    opt = KfacOptimizer(layers, cfg, n, rng_seed=seed)
    xs = []
    for L in layers:
        xs += [np.eye(L.dim_a), np.eye(L.dim_g)]
    cached = None
    for k in range(2):
        a_m, g_m, grads = [], [], []
        for l, L in enumerate(layers):
            a, _ = port.sample_gaussian(port.substream(3, k, 2 * l), 0, L.dim_a, n)
            g, _ = port.sample_gaussian(port.substream(3, k, 2 * l + 1), 0, L.dim_g, n)
            j, _ = port.sample_gaussian(port.substream(4, k, l), 0, L.dim_g, L.dim_a)
            a_m.append(a); g_m.append(g); grads.append(j)
            xs[2 * l] = port.ea_update(xs[2 * l], a / math.sqrt(n), 0.95)
            xs[2 * l + 1] = port.ea_update(xs[2 * l + 1], g / math.sqrt(n), 0.95)
        opt.accumulate_factors([t32(a, cuda) for a in a_m], [t32(g, cuda) for g in g_m])
        outs = opt.step([t32(j, cuda) for j in grads], step=k)
        if k == 0:  # step 0 % T_KI == 0: decompose; step 1 reuses the cached decompositions
            cached = []
            for f, x in enumerate(xs):
                if method == "kfac":
                    pm, dv = port.sym_eig(x)
                    cached.append((pm, dv))
                else:
                    fn = port.srevd if method == "sre" else port.rsvd_psd
                    u0, d0, _ = fn(x, r, p, q, port.substream(seed, k, f), 0)
                    cached.append((u0, d0))
        for l in range(len(layers)):
            (ua, da), (ug, dg) = cached[2 * l], cached[2 * l + 1]
            if method == "kfac":
                m = port.apply_eig_damped_inverse(ua, da, lam, grads[l], "right")
                s0 = port.apply_eig_damped_inverse(ug, dg, lam, m, "left")
            else:
                s0 = port.precondition(ua, da, ug, dg, lam, grads[l])
            assert rel_fro(np64(outs[l]), s0) < TOL, (k, l)
    assert opt.timings.decomposition > 0 and opt.timings.inverse_apply > 0


def test_spectrum_snapshot_matches_oracle(port, cuda):
    """kfactor.hpp:56-63 spectrum on the device factor vs the oracle's sym_eig (clamped at 0)."""
    from paper_2206_15397_b200.kfac import spectrum

    x = build_factor(port, 200, 64, 5, 1.0, f=0)
    _, d0 = port.sym_eig(x)
    rep = spectrum(t32(x, cuda))
    ev = np.asarray(rep.eigenvalues)
    top = np.maximum(d0, 0.0)[:40]
    assert eig_err(ev[:40], top) < TOL and rep.lambda_max == pytest.approx(top[0], rel=1e-6)


# ------------------------------------------------------------------------- general rsvd (rnla.hpp:62-77)
@pytest.mark.skipif(not __import__("oracle").ref_available(), reason="oracle/_ref (the reference build) not present")
@pytest.mark.parametrize("rows,cols", [(300, 200), (200, 300), (517, 517)])
def test_rsvd_general_matches_reference(port, cuda, rows, cols):
    """SvdResult rsvd on a rectangular matrix with a geometric spectrum vs the reference's own rsvd on the same input
    and Omega stream: singular values, the sign-invariant product U diag(s) V^T, orthonormality, counter advance."""
    import oracle
    import paper_2206_15397_b200 as rk

    ref = oracle.ref()
    k = min(rows, cols)
    g1, _ = port.sample_gaussian(41, 0, rows, k)
    g2, _ = port.sample_gaussian(42, 0, cols, k)
    u0, _ = port.qr_thin(g1)
    v0, _ = port.qr_thin(g2)
    x = ((u0 * geometric_spectrum(k, 0.9)[None, :]) @ v0.T).astype(np.float32).astype(np.float64)
    r, p, q = 20, 5, 2
    seed = port.substream(OMEGA_ROOT, 0, 5)
    ur, sr, vr, cr = ref.rsvd(x, r, p, q, seed, 0)
    rng = rk.RngState(seed, 0)
    res = rk.rsvd(t32(x, cuda), rk.SketchParams(r, p, q), rng)
    assert rng.counter == cr
    u1, s1, v1 = np64(res.u), np64(res.s), np64(res.v)
    assert u1.shape == ur.shape and v1.shape == vr.shape
    assert eig_err(s1, sr) < TOL
    assert rel_fro((u1 * s1) @ v1.T, (ur * sr) @ vr.T) < TOL
    assert orth_err(u1) < 1e-5 and orth_err(v1) < 1e-5
