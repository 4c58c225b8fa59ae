"""Multi-GPU host logic on CPU: LPT layer sharding and the single packed all-gather (gloo, world_size 2).  The
gathered result must be bitwise identical to the 1-rank result (BASELINE config 4)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_15397_b200.partition import (GatherLayout, all_gather_results, layer_cost, lpt_partition, makespan,
                                             sketch_width)

VGG_A = [28, 577, 577, 1153, 1153, 2305, 2305, 2305, 4609, 4609, 4609, 4609, 4609, 513, 513, 513]
VGG_G = [64, 64, 128, 128, 256, 256, 256, 512, 512, 512, 512, 512, 512, 512, 512, 10]


def test_sketch_width_matches_clamp_sketch():
    # rnla.hpp:35-43
    assert sketch_width(28, 220, 10) == 28
    assert sketch_width(4609, 220, 10) == 230
    assert sketch_width(225, 220, 10) == 225
    assert sketch_width(10, 220, 10) == 10


def test_lpt_partition_is_deterministic_and_complete():
    costs = [layer_cost(a, g, 220, 10) for a, g in zip(VGG_A, VGG_G)]
    for n in (1, 2, 4, 8):
        parts = lpt_partition(costs, n)
        assert parts == lpt_partition(costs, n)
        assert sorted(i for p in parts for i in p) == list(range(16))
    ideal = sum(costs)
    # layer-granularity LPT ceilings 1.99 / 2.99 / 5.98x on 2/4/8 ranks
    for n, lo in ((2, 1.98), (4, 2.95), (8, 5.9)):
        assert ideal / makespan(costs, lpt_partition(costs, n)) >= lo


def test_gather_layout_roundtrip():
    sizes = [3, 5, 2, 7]
    parts = [[0, 3], [1, 2]]
    lay = GatherLayout.build(sizes, parts)
    assert lay.chunk == 10
    buf = torch.arange(2 * lay.chunk, dtype=torch.float32)
    for l in range(4):
        off = lay.global_offset(l)
        assert 0 <= off and off + sizes[l] <= 2 * lay.chunk


def _layer_result(l, shape):
    g = torch.Generator().manual_seed(1000 + l)
    return torch.randn(*shape, generator=g)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shapes = [(g, a) for a, g in zip(VGG_A[:6], VGG_G[:6])]
    costs = [layer_cost(a, g, 220, 10) for a, g in zip(VGG_A[:6], VGG_G[:6])]
    parts = lpt_partition(costs, world)
    lay = GatherLayout.build([a * g for a, g in zip(VGG_A[:6], VGG_G[:6])], parts)
    local = {l: _layer_result(l, shapes[l]) for l in parts[rank]}
    views, _ = all_gather_results(lay, rank, local, shapes)
    ok = all(torch.equal(views[l], _layer_result(l, shapes[l])) for l in range(6))
    q.put((rank, ok))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(120)
def test_all_gather_two_ranks_gloo_bitwise():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in procs]
    for p in procs:
        p.join(timeout=30)
    assert sorted(res) == [(0, True), (1, True)]


# ---- the sharded STEP through the collective: every rank runs its LPT shard of the preconditioned
# step (EA -> srevd -> RIGHT_A / LEFT_G, optimizer.hpp:139-167) with the global factor tags as substream ids, the
# packed outputs are all-gathered over gloo, and the gathered step equals the single-process step bitwise.  The
# per-layer arithmetic is the CPU oracle's (the GPU kernels' own shard bitwise-equality is
# tests/test_gpu_configs.py::test_config4_sharded_step_is_bitwise_the_one_gpu_step).
STEP_LAYERS = [(28, 64), (65, 32), (49, 10), (33, 40), (17, 12)]
STEP_R, STEP_P, STEP_Q, STEP_N, STEP_LAM = 8, 4, 1, 16, 0.1


def _oracle_layer_step(port, l):
    """Layer l of the reference step with global tags: factors 2l (A) and 2l+1 (G)."""
    import numpy as np

    a, g = STEP_LAYERS[l]
    decs = []
    for which, d in enumerate((a, g)):
        f = 2 * l + which
        x = np.zeros((d, d))
        for k in range(3):
            x = port.ea_update(x, port.synthetic_m(220615397, k, f, STEP_N, d, 1.0), 0.95)
        u, dv, _ = port.srevd(x, STEP_R, STEP_P, STEP_Q, port.substream(7, 0, f), 0)
        decs.append((u, dv))
    j, _ = port.sample_gaussian(port.substream(99, l, 0), 0, g, a)
    return port.precondition(decs[0][0], decs[0][1], decs[1][0], decs[1][1], STEP_LAM, j)


def _step_worker(rank, world, port_no, q):
    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    port = oracle.port()
    shapes = [(g, a) for a, g in STEP_LAYERS]
    costs = [layer_cost(a, g, STEP_R, STEP_P) for a, g in STEP_LAYERS]
    parts = lpt_partition(costs, world)
    lay = GatherLayout.build([a * g for a, g in STEP_LAYERS], parts)
    local = {l: torch.as_tensor(_oracle_layer_step(port, l), dtype=torch.float32) for l in parts[rank]}
    views, _ = all_gather_results(lay, rank, local, shapes)
    full = [torch.as_tensor(_oracle_layer_step(port, l), dtype=torch.float32) for l in range(len(STEP_LAYERS))]
    q.put((rank, all(torch.equal(views[l], full[l]) for l in range(len(STEP_LAYERS))), [len(p) for p in parts]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_sharded_step_gathered_over_gloo_equals_the_single_process_step():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_step_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=150) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    assert [r[:2] for r in res] == [(0, True), (1, True)]
    assert all(n >= 1 for n in res[0][2])  # both ranks own layers
