"""GPU counterpart of the reference's bench-inverse (harness.hpp:402-478): median time of exact K-FAC inversion
(full eigendecomposition + apply_eig_damped_inverse) vs rand-EVD (srevd / rsvd_psd, r=220, p=10, q=4) + the
damped low-rank apply, on the same random PSD matrices (g g^T / cols + 0.01 I), and the log-log slopes in d.

    python tools/bench_inverse.py [--dims 512 1024 2048 4096] [--reps 5] > profiles/rNN_bench_inverse.json
"""
import argparse
import json
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2206_15397_b200 as rk

    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs="+", default=[512, 1024, 2048, 4096])
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    lam, sk = 0.1, rk.SketchParams(220, 10, 4)
    gen = torch.Generator(device="cuda").manual_seed(0xBE7C)
    med = {"exact": {}, "rsvd": {}, "srevd": {}}
    for d in a.dims:
        g = torch.randn(d, min(d, 512), device="cuda", generator=gen)
        x = g @ g.T / g.shape[1] + 0.01 * torch.eye(d, device="cuda")
        v = torch.randn(d, d, device="cuda", generator=gen)

        def exact():
            return rk.apply_eig_damped_inverse(rk.sym_eig(x), lam, v, rk.ApplySide.LEFT)

        def rsvd(rep):
            return rk.apply_lowrank_damped_inverse(rk.rsvd_psd(x, sk, rk.RngState(rk.substream_seed(7, d, 2 * rep))),
                                                   lam, v, rk.ApplySide.LEFT)

        def srevd(rep):
            return rk.apply_lowrank_damped_inverse(rk.srevd(x, sk, rk.RngState(rk.substream_seed(7, d, 2 * rep + 1))),
                                                   lam, v, rk.ApplySide.LEFT)

        for name, fn in (("exact", lambda rep: exact()), ("rsvd", rsvd), ("srevd", srevd)):
            fn(0)  # warm-up (plan / solver workspaces)
            ts = []
            for rep in range(a.reps):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn(rep)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / 1e3)
            med[name][d] = statistics.median(ts)
    slopes = {}
    for name, series in med.items():
        xs = [math.log(d) for d in series]
        ys = [math.log(t) for t in series.values()]
        n = len(xs)
        sx, sy = sum(xs), sum(ys)
        sxx = sum(x * x for x in xs)
        sxy = sum(x * y for x, y in zip(xs, ys))
        slopes[name] = (n * sxy - sx * sy) / (n * sxx - sx * sx) if n > 1 else None
    print(json.dumps({"what": "bench-inverse on one B200 (harness.hpp:402-478 construction; exact = this repo's FP64 "
                      "eigensolver csrc/symeig.cu (Householder + divide and conquer) + our apply kernels; rsvd/srevd = "
                      "our rand-EVD + apply)", "lambda": lam,
                      "sketch": [220, 10, 4], "median_seconds": med, "loglog_slopes": slopes}))


if __name__ == "__main__":
    main()
