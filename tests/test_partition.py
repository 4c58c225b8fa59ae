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
