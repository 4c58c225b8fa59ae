"""CUDA-graph replays of the step (the bench's e2e path): bitwise the eager calls."""
import math

import pytest

pytestmark = pytest.mark.gpu


def test_host_step_graph_is_bitwise_step_host(cuda):
    """rk.HostStepGraph (step_host captured once: pinned H2D copies, every group's chain, D2H) == step_host."""
    import torch
    import paper_2206_15397_b200 as rk

    layers = [rk.LayerSpec(577, 64), rk.LayerSpec(300, 257), rk.LayerSpec(28, 64), rk.LayerSpec(513, 10)]
    st = rk.StreamedStep(layers, groups=2, rank=40, oversampling=10, power_iters=2, n_samples=[64], device=0)
    g = torch.Generator(device="cuda").manual_seed(9)
    h_samples, h_grads = [], []
    for d in st.dims:
        s = torch.arange(1, d + 1, device=cuda, dtype=torch.float32).pow(-1.0)
        h_samples.append((torch.randn(d, 64, device=cuda, generator=g) * s[:, None] / math.sqrt(64)).cpu().pin_memory())
    for L in layers:
        h_grads.append(torch.randn(L.dim_g, L.dim_a, device=cuda, generator=g).cpu().pin_memory())
    h_outs = [torch.empty(L.dim_g, L.dim_a).pin_memory() for L in layers]
    x0 = [x.clone() for x in st.factors]

    def reset():
        for x, y in zip(st.factors, x0):
            x.copy_(y)

    reset()
    st.step_host(7, 0, 0.1, h_samples, h_grads, h_outs)
    torch.cuda.synchronize()
    eager = [o.clone() for o in h_outs]
    reset()
    graph = rk.HostStepGraph(st, 7, 0, 0.1, h_samples, h_grads, h_outs)
    for _ in range(2):  # replays start from the restored factors, like the bench
        reset()
        for o in h_outs:
            o.zero_()
        graph.replay()
        torch.cuda.synchronize()
        for a, b in zip(h_outs, eager):
            assert torch.equal(a, b)
    assert graph.launches > 0


def test_step_graph_replays_take_their_omega_seed_at_replay_time(cuda):
    """One captured step serves every step id: replay(rng_root, step) == the eager step(rng_root, step), bitwise
    (the captured Omega kernel reads (root, step) from a pinned host pair, rkfac_plan_set_step_seed)."""
    import torch
    import paper_2206_15397_b200 as rk

    layers = [rk.LayerSpec(577, 64), rk.LayerSpec(300, 257), rk.LayerSpec(513, 10)]
    st = rk.StreamedStep(layers, groups=2, rank=40, oversampling=10, power_iters=2, n_samples=[64], device=0)
    g = torch.Generator(device="cuda").manual_seed(11)
    for f, d in enumerate(st.dims):
        s = torch.arange(1, d + 1, device=cuda, dtype=torch.float32).pow(-1.0)
        st.samples[f].copy_(torch.randn(d, 64, device=cuda, generator=g) * s[:, None] / math.sqrt(64))
    for l, L in enumerate(layers):
        st.grads[l].copy_(torch.randn(L.dim_g, L.dim_a, device=cuda, generator=g))
    x0 = [x.clone() for x in st.factors]

    def reset():
        for x, y in zip(st.factors, x0):
            x.copy_(y)

    eager = {}
    for root, step in ((7, 0), (7, 5), (9, 2)):
        reset()
        st.step(root, step, 0.1)
        torch.cuda.synchronize()
        eager[(root, step)] = [o.clone() for o in st.outs] + [st.lowrank(f).d.clone() for f in range(len(st.dims))]
    assert not torch.equal(eager[(7, 0)][0], eager[(7, 5)][0])  # different Omega, different randomized answer
    reset()
    graph = rk.StepGraph(st, 7, 0, 0.1)
    for key in ((7, 5), (9, 2), (7, 0)):
        reset()
        graph.replay(*key)
        torch.cuda.synchronize()
        got = [o.clone() for o in st.outs] + [st.lowrank(f).d.clone() for f in range(len(st.dims))]
        for a, b in zip(got, eager[key]):
            assert torch.equal(a, b), key
