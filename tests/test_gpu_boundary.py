"""The drop-in boundary on the GPU: the single-factor C-ABI operators run the same tcgen05
stages as the batched plan (bitwise), and the multi-GPU collective is reachable through the C-ABI (a single-rank NCCL
clique: rkfac_nccl_unique_id -> rkfac_nccl_init -> rkfac_allgather / rkfac_plan_set_gather + rkfac_plan_step)."""
import math

import numpy as np
import pytest

from tests.helpers import GRAD_ROOT, OMEGA_ROOT, ROOT_SEED

pytestmark = pytest.mark.gpu


def _filled_step(rk, cuda, port, layers, n=128, steps=3):
    import torch

    st = rk.BatchedStep(layers, rank=40, oversampling=10, power_iters=2, method=rk.DecompMethod.SREVD,
                        n_samples=[n], device=0)
    st.set_ea_lo_mode(0)  # the single-factor EA forms the lo planes in smem, as here
    for k in range(steps):
        for f, d in enumerate(st.dims):
            st.samples[f].copy_(torch.as_tensor(port.synthetic_m(ROOT_SEED, k, f, n, d, 1.0), dtype=torch.float32,
                                                device=cuda))
        st.ea_update(0.95, 1.0)
    for l, L in enumerate(layers):
        st.grads[l].copy_(rk.sample_gaussian(rk.RngState(rk.substream_seed(GRAD_ROOT, l, 0)), L.dim_g, L.dim_a,
                                             device=cuda))
    return st


def test_single_factor_ea_is_bitwise_the_plan_ea(port, cuda):
    """rkfac_ea_update (cached tcgen05 stage) == the plan's grouped EA, factor by factor, incl. a factor whose pitch
    is not a TMA stride (d = 577: padded-copy path)."""
    import torch
    import paper_2206_15397_b200 as rk

    layers = [rk.LayerSpec(577, 1153)]
    n = 128
    st = rk.BatchedStep(layers, rank=40, oversampling=10, power_iters=2, n_samples=[n], device=0)
    st.set_ea_lo_mode(0)
    singles = [rk.EAKFactor.create(d, 0.95, zero_init=True, device=cuda) for d in st.dims]
    for k in range(3):
        ms = []
        for f, d in enumerate(st.dims):
            m = torch.as_tensor(port.synthetic_m(ROOT_SEED, k, f, n, d, 1.0), dtype=torch.float32, device=cuda)
            st.samples[f].copy_(m)
            ms.append(m)
        st.ea_update(0.95, 1.0)
        for f in range(len(st.dims)):
            rk.ea_update(singles[f], ms[f])
    torch.cuda.synchronize()
    for f in range(len(st.dims)):
        assert torch.equal(singles[f].mbar, st.factors[f]), f


def test_single_factor_apply_chain_is_bitwise_the_plan_precondition(port, cuda):
    """RIGHT_A then LEFT_G through rkfac_apply_lowrank_damped_inverse == the plan's batched preconditioning."""
    import torch
    import paper_2206_15397_b200 as rk

    layers = [rk.LayerSpec(577, 300), rk.LayerSpec(64, 10)]
    st = _filled_step(rk, cuda, port, layers)
    st.decompose(OMEGA_ROOT, 0)
    st.precondition(0.1)
    torch.cuda.synchronize()
    for l in range(len(layers)):
        mid = rk.apply_lowrank_damped_inverse(st.lowrank(2 * l), 0.1, st.grads[l], rk.ApplySide.RIGHT)
        out = rk.apply_lowrank_damped_inverse(st.lowrank(2 * l + 1), 0.1, mid, rk.ApplySide.LEFT)
        torch.cuda.synchronize()
        assert torch.equal(out, st.outs[l]), l


def test_single_factor_ops_are_asynchronous_and_cached(port, cuda):
    """A repeated call with the same operands enqueues only its kernels: no new stage is built (the cached stage's
    launch count per call stays constant) and the result is reproducible."""
    import torch
    import paper_2206_15397_b200 as rk

    d, n = 512, 128
    f = rk.EAKFactor.create(d, 0.95, device=cuda)
    m = torch.as_tensor(port.synthetic_m(ROOT_SEED, 0, 0, n, d, 1.0), dtype=torch.float32, device=cuda)
    ctx = rk.context()
    rk.ea_update(f, m)
    n0 = ctx.launches()
    rk.ea_update(f, m)
    n1 = ctx.launches()
    rk.ea_update(f, m)
    n2 = ctx.launches()
    assert n1 - n0 == n2 - n1 == 1  # one tcgen05 launch per cached EA call (aligned operands: no copies)


def test_nccl_single_rank_clique_through_the_c_abi(cuda):
    import torch
    import paper_2206_15397_b200 as rk

    ctx = rk.context()
    uid = rk.nccl_unique_id()
    assert len(uid) == 128
    ctx.nccl_init(uid, 1, 0)
    send = torch.randn(1000, device=cuda)
    recv = torch.empty(1000, device=cuda)
    ctx.allgather(send, recv)
    torch.cuda.synchronize()
    assert torch.equal(send, recv)


def test_plan_step_ends_with_the_all_gather(port, cuda):
    """rkfac_plan_set_gather: the step packs this rank's outputs into its chunk and all-gathers (one rank here)."""
    import torch
    import paper_2206_15397_b200 as rk

    ctx = rk.context()
    if getattr(ctx, "nranks", None) is None:
        ctx.nccl_init(rk.nccl_unique_id(), 1, 0)
    layers = [rk.LayerSpec(300, 64), rk.LayerSpec(28, 10)]
    st = _filled_step(rk, cuda, port, layers)
    sizes = [L.dim_a * L.dim_g for L in layers]
    offsets = [0, sizes[0] + 7]  # any layout inside the chunk
    chunk = offsets[1] + sizes[1] + 5
    gathered = torch.full((chunk,), float("nan"), device=cuda)
    st.set_gather(chunk, offsets, gathered)
    st.step(OMEGA_ROOT, 0, 0.1)
    torch.cuda.synchronize()
    for l in range(len(layers)):
        assert torch.equal(gathered[offsets[l]:offsets[l] + sizes[l]], st.outs[l].reshape(-1)), l
    assert st.workspace_bytes() > 0


def test_step_overlap_and_ea_decompose_are_bitwise_the_separate_calls(port, cuda, monkeypatch):
    """rkfac_plan_step / rkfac_plan_ea_decompose run Omega (and the gradient copy, U^T's copy-out) on the plan's side
    stream next to the EA update / the preconditioning; the results are bitwise those of ea_update -> decompose ->
    precondition issued one after the other, with the overlap on (default here) and forced off."""
    import torch
    import paper_2206_15397_b200 as rk

    layers = [rk.LayerSpec(577, 128), rk.LayerSpec(300, 64)]

    def run(mode, overlap):
        monkeypatch.setenv("RKFAC_STEP_OVERLAP", "1" if overlap else "0")
        st = _filled_step(rk, cuda, port, layers)
        if mode == "step":
            st.step(OMEGA_ROOT, 3, 0.1, 0.95, 1.0)
        elif mode == "ea_decompose":
            st.ea_decompose(OMEGA_ROOT, 3, 0.95, 1.0)
            st.precondition(0.1)
        else:
            st.ea_update(0.95, 1.0)
            st.decompose(OMEGA_ROOT, 3)
            st.precondition(0.1)
        torch.cuda.synchronize()
        return ([x.clone() for x in st.factors], [st.lowrank(f).u.clone() for f in range(len(st.dims))],
                [st.lowrank(f).d.clone() for f in range(len(st.dims))], [o.clone() for o in st.outs])

    ref = run("separate", False)
    for mode in ("step", "ea_decompose"):
        for overlap in (True, False):
            got = run(mode, overlap)
            for a, b in zip(ref, got):
                for x, y in zip(a, b):
                    assert torch.equal(x, y), (mode, overlap)


def test_overlapped_power_iteration_option_meets_the_bar_at_config1(port, cuda):
    """rkfac_plan_set_overlap (opt-in: the product X Y next to Gram + Cholesky-inverse, Y' = (X Y) L^-T) reproduces the
    reference's config-1 decomposition within the 1e-4 bar; it is off by default because config 5's spectrum
    (lambda_r / lambda_1 = 1.6e-6) moves the last Ritz values by 3e-4, which
    overlap_error_estimate predicts from a previous decomposition's eigenvalues."""
    import torch
    import paper_2206_15397_b200 as rk

    d, n, r, p, q = 512, 256, 64, 10, 2
    x = np.zeros((d, d))
    for k in range(20):
        x = port.ea_update(x, port.synthetic_m(ROOT_SEED, k, 0, n, d, 1.0), 0.95)
    seed = port.substream(OMEGA_ROOT, 0, 0)
    u0, d0, _ = port.srevd(x, r, p, q, seed, 0)
    xt = torch.as_tensor(x, dtype=torch.float32, device=cuda)
    st = rk.BatchedStep([rk.LayerSpec(d, d)], rank=r, oversampling=p, power_iters=q, method=rk.DecompMethod.SREVD,
                        device=0)
    st.set_overlap(True)
    st.factors[0].copy_(xt)
    st.factors[1].copy_(xt)
    st.decompose(OMEGA_ROOT, 0)
    torch.cuda.synchronize()
    lr = st.lowrank(0)
    u1, d1 = lr.u.double().cpu().numpy(), lr.d.double().cpu().numpy()
    rec0, rec1 = (u0 * d0) @ u0.T, (u1 * d1) @ u1.T
    assert np.linalg.norm(rec1 - rec0) / np.linalg.norm(rec0) < 1e-4
    assert np.max(np.abs(d1 - d0) / d0) < 1e-4
    assert rk.overlap_error_estimate(lr.d) < 1e-4  # lambda_r / lambda_1 ~ 1/64^2 here: far inside the safe range
