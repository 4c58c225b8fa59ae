"""Multi-GPU sharding of the batched step.

Layers are independent units: layer l's EA updates, both rand-EVDs and its preconditioning touch only its own two
factors (optimizer.hpp:147-165).  So layers are assigned whole to ranks (both factors of a layer on the owning GPU)
by LPT on the decomposition cost c_l = d_A^2 w_A + d_G^2 w_G (proportional to the (2q+2) X*Q products), and the
only collective is one all-gather of the preconditioned gradients.  Factor tags stay global (2l + which), so every
Omega is the one the 1-GPU run draws and the gathered result is bitwise identical to the 1-GPU result.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence


def sketch_width(d: int, r: int, p: int) -> int:
    """rnla.hpp:35-43 clamp_sketch: w = min(r, d) + clamped p."""
    if r > d:
        return d
    return min(r + p, d)


def layer_cost(dim_a: int, dim_g: int, r: int, p: int) -> float:
    return float(dim_a) ** 2 * sketch_width(dim_a, r, p) + float(dim_g) ** 2 * sketch_width(dim_g, r, p)


def lpt_partition(costs: Sequence[float], nranks: int) -> List[List[int]]:
    """Longest-processing-time-first: biggest layer to the least-loaded rank (ties -> lowest rank, then lowest
    layer index), deterministic.  Returns per-rank sorted layer lists."""
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    loads = [0.0] * nranks
    parts: List[List[int]] = [[] for _ in range(nranks)]
    for i in order:
        k = min(range(nranks), key=lambda j: (loads[j], j))
        parts[k].append(i)
        loads[k] += costs[i]
    return [sorted(p) for p in parts]


def makespan(costs: Sequence[float], parts: Sequence[Sequence[int]]) -> float:
    return max((sum(costs[i] for i in p) for p in parts), default=0.0)


@dataclass
class GatherLayout:
    """Packed uniform-chunk all-gather: rank k's layers are concatenated (row-major d_G x d_A each) into a chunk
    padded to the largest rank payload, so a single ncclAllGather moves everything."""

    parts: List[List[int]]
    sizes: List[int]          # elements per layer
    chunk: int                # padded elements per rank
    offsets: List[int]        # offset of layer l inside its owner's chunk
    owner: List[int]          # rank owning layer l

    @staticmethod
    def build(sizes: Sequence[int], parts: Sequence[Sequence[int]]) -> "GatherLayout":
        owner = [-1] * len(sizes)
        offsets = [0] * len(sizes)
        chunk = 0
        for k, p in enumerate(parts):
            off = 0
            for l in p:
                owner[l] = k
                offsets[l] = off
                off += sizes[l]
            chunk = max(chunk, off)
        if any(o < 0 for o in owner):
            raise ValueError("a layer is not assigned to any rank")
        return GatherLayout([list(p) for p in parts], list(sizes), chunk, offsets, owner)

    def global_offset(self, l: int) -> int:
        return self.owner[l] * self.chunk + self.offsets[l]


def pack_local(layout: GatherLayout, rank: int, tensors, out):
    """Copies this rank's layer results (dict layer -> tensor) into its chunk `out` (1-D, length chunk)."""
    for l in layout.parts[rank]:
        n = layout.sizes[l]
        out[layout.offsets[l]:layout.offsets[l] + n].copy_(tensors[l].reshape(-1))


def unpack_all(layout: GatherLayout, gathered, shapes):
    """Views of every layer's result inside the gathered buffer (world * chunk)."""
    res = []
    for l, shp in enumerate(shapes):
        off = layout.global_offset(l)
        res.append(gathered[off:off + layout.sizes[l]].view(*shp))
    return res


def all_gather_results(layout: GatherLayout, rank: int, local, shapes, group=None):
    """One all-gather (NCCL on GPU, gloo in the CPU tests) of the per-rank packed results."""
    import torch
    import torch.distributed as dist

    world = len(layout.parts)
    dev = next(iter(local.values())).device if local else torch.device("cpu")
    send = torch.zeros(layout.chunk, dtype=torch.float32, device=dev)
    pack_local(layout, rank, local, send)
    recv = torch.empty(world * layout.chunk, dtype=torch.float32, device=dev)
    if world == 1:
        recv.copy_(send)
    else:
        dist.all_gather_into_tensor(recv, send, group=group)
    return unpack_all(layout, recv, shapes), recv
