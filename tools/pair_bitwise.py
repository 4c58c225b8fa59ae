#!/usr/bin/env python
"""Stress check of the CTA-pair X*Q kernel: the VGG16 step's outputs hashed over repeated steps.  Run once with
RKFAC_XQ_PAIR=1 and once with RKFAC_XQ_PAIR=0 (the single-CTA kernels): every hash must agree -- the pair kernel
keeps each element's K order, so any difference is a synchronisation bug (a stale operand read).
usage: python tools/pair_bitwise.py [reps] [groups] [vgg16|mixed] -> one line per repetition: sha256 of all U^T,
eigenvalues and outputs ("mixed": many mid-size factors with dimensions off every tile boundary, rank 96)"""
import hashlib
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2206_15397_b200 as rk  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    groups = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    which = sys.argv[3] if len(sys.argv) > 3 else "vgg16"
    if which == "mixed":  # enough 256-row tiles to stay on the pair kernel, none of them aligned
        dims = [130, 257, 300, 511, 640, 1000, 1153, 1290, 1535, 2049, 2305, 777, 897, 1025, 385, 129]
        layers = [(dims[i], dims[(i + 5) % len(dims)]) for i in range(len(dims))]
        n, e, r, p, q, lam = 96, 1.0, 96, 10, 2, 0.1
    else:
        layers, n, e, r, p, q, lam, _ = bench.WORKLOADS["vgg16"]
    dev = torch.device("cuda", 0)
    specs = [rk.LayerSpec(a, g) for a, g in layers]
    if groups > 1:
        st = rk.StreamedStep(specs, groups=groups, rank=r, oversampling=p, power_iters=q, n_samples=[n], device=0)
    else:
        st = rk.BatchedStep(specs, rank=r, oversampling=p, power_iters=q, n_samples=[n], device=0)
    for f, d in enumerate(st.dims):
        z = rk.sample_gaussian(rk.RngState(rk.substream_seed(bench.ROOT_SEED, 0, f)), n, d, device=dev)
        s = torch.arange(1, d + 1, device=dev, dtype=torch.float64).pow(-e)
        st.samples[f].copy_((z.double() * s[None, :] / math.sqrt(n)).t().float())
    for l, (a, g) in enumerate(layers):
        st.grads[l].copy_(rk.sample_gaussian(rk.RngState(rk.substream_seed(bench.GRAD_ROOT, l, 0)), g, a, device=dev))
    for k in range(reps):
        st.step(bench.OMEGA_ROOT, k, lam)
        torch.cuda.synchronize()
        h = hashlib.sha256()
        for f in range(len(st.dims)):
            h.update(st.bases_t[f].contiguous().cpu().numpy().tobytes())
            h.update(st.dvals[f].cpu().numpy().tobytes())
        for o in st.outs:
            h.update(o.contiguous().cpu().numpy().tobytes())
        print(k, h.hexdigest(), flush=True)


if __name__ == "__main__":
    main()
