#!/usr/bin/env python
"""Where the end-to-end step's time goes: StreamedStep.step_host (the bench's e2e call) with per-group events
(samples in, decomposed, preconditioned, results out), median over steps, in ms from the fork.

    python tools/e2e_timeline.py [--groups 5] [--steps 10]
"""
import argparse
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import paper_2206_15397_b200 as rk

    ap = argparse.ArgumentParser()
    ap.add_argument("--groups", type=int, default=5)
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    layers, n, e, r, p, q, lam, warm = bench.WORKLOADS["vgg16"]
    specs = [rk.LayerSpec(x, y) for x, y in layers]
    st = rk.StreamedStep(specs, groups=a.groups, rank=r, oversampling=p, power_iters=q, n_samples=[n], device=0)
    dev = torch.device("cuda", 0)
    for k in range(warm + 1):
        for f, d in enumerate(st.dims):
            z = rk.sample_gaussian(rk.RngState(rk.substream_seed(bench.ROOT_SEED, k, f)), n, d, device=dev)
            s = torch.arange(1, d + 1, device=dev, dtype=torch.float64).pow(-e)
            st.samples[f].copy_((z.double() * s[None, :] / math.sqrt(n)).t().float())
        if k < warm:
            st.ea_update(0.95, 1.0)
    for l, (x, y) in enumerate(layers):
        st.grads[l].copy_(rk.sample_gaussian(rk.RngState(rk.substream_seed(bench.GRAD_ROOT, l, 0)), y, x, device=dev))
    h_samples = [x.cpu().pin_memory() for x in st.samples]
    h_grads = [x.cpu().pin_memory() for x in st.grads]
    h_outs = [torch.empty_like(x, device="cpu").pin_memory() for x in st.outs]
    x0 = [x.clone() for x in st.factors]
    rows = {}
    for i in range(3 + a.steps):
        for x, y in zip(st.factors, x0):
            x.copy_(y)
        tl = []
        st.step_host(bench.OMEGA_ROOT, 0, lam, h_samples, h_grads, h_outs, 0.95, 1.0, timeline=tl)
        torch.cuda.synchronize()
        if i < 3:
            continue
        fork = tl[0][1]
        for name, ev in tl[1:]:
            rows.setdefault(name, []).append(fork.elapsed_time(ev))
    print("groups (layers):", [list(p) for p in st.parts])
    for name in sorted(rows, key=lambda k: statistics.median(rows[k])):
        print(f"{statistics.median(rows[name]):8.3f} ms  {name}")


if __name__ == "__main__":
    main()
