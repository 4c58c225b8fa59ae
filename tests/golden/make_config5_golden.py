"""Generates tests/golden/config5_golden.npz from the REFERENCE itself (oracle/_ref: the unmodified reference headers
compiled by oracle/Makefile) for BASELINE config 5 -- one factor pair at d = 16384.  Run in the build container
(about 30 min on 2 threads; the reference is single-threaded FP64 scalar code):

    python tests/golden/make_config5_golden.py

Inputs (all from the reference RNG, rng.hpp:13-63):
  * factor f in {0 (A), 1 (G)}: zero-init EA (rho = 0.95) over 10 steps of M = X^T / sqrt(n), X = Z diag(s),
    Z = sample_gaussian(RngState(220615397).substream(k, f), n = 512, d), s_i = i^-1.2  (kfactor.hpp:33-41 ea_update)
  * srevd with r = 256, p = 16, q = 4, Omega from RngState(7).substream(0, f)          (rnla.hpp:90-105)
  * J = sample_gaussian(RngState(99).substream(0, 0), d, d), lambda = 0.05
    S = LEFT_G(RIGHT_A(J))                                                             (optimizer.hpp:159-162)

The full matrices are 2 GiB each in FP64, so the fixture keeps size-independent witnesses: the top-r eigenvalues,
and fixed random projections (sketch vectors V, W drawn from the reference RNG, seeds below) of the factor X, the
sign-invariant projector U diag(d) U^T and the preconditioned gradient S: X V, U diag(d) U^T V, S V and W^T S
(stored as FP32: 6e-8 relative, far below the 1e-4 bar), plus Frobenius norms.  A projection onto 3 Gaussian vectors preserves a relative error to within a small factor, so
comparing sketches at 1e-4 checks the full matrices at that bar.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

ROOT_SEED, OMEGA_ROOT, GRAD_ROOT = 220615397, 7, 99
D, N, E, STEPS, RHO = 16384, 512, 1.2, 10, 0.95
R, P, Q, LAM = 256, 16, 4, 0.05
SKETCH_SEED_V, SKETCH_SEED_W, NSK = 5150001, 5150002, 3
OUT = os.path.join(HERE, "config5_golden.npz")


def sketch_vectors(port):
    v, _ = port.sample_gaussian(SKETCH_SEED_V, 0, D, NSK)
    w, _ = port.sample_gaussian(SKETCH_SEED_W, 0, D, NSK)
    return v, w


def main():
    if not oracle.ref_available():
        raise SystemExit("oracle/_ref not built (needs /root/reference): run `make -C oracle`")
    ref = oracle.ref()
    port = oracle.port()
    t0 = time.time()

    def build(f):
        x = np.zeros((D, D))
        for k in range(STEPS):
            m = port.synthetic_m(ROOT_SEED, k, f, N, D, E)  # bit-pinned to the reference RNG (tests/test_oracle.py)
            x = ref.ea_update(x, m, RHO)
            print(f"factor {f}: EA step {k} done at {time.time() - t0:.0f}s", flush=True)
        u, dv, _ = ref.srevd(x, R, P, Q, ref.substream(OMEGA_ROOT, 0, f), 0)
        print(f"factor {f}: srevd done at {time.time() - t0:.0f}s", flush=True)
        return x, u, dv

    (xa, ua, da), (xg, ug, dg) = oracle.parallel_map(build, [0, 1], 2)
    v, w = sketch_vectors(port)
    out = {"dims": np.array([D, N, STEPS, R, P, Q]), "params": np.array([E, RHO, LAM])}
    for tag, x, u, dv in (("a", xa, ua, da), ("g", xg, ug, dg)):
        out[f"dvals_{tag}"] = dv
        out[f"xv_{tag}"] = (x @ v).astype(np.float32)
        out[f"pv_{tag}"] = (u @ (dv[:, None] * (u.T @ v))).astype(np.float32)
        out[f"xnorm_{tag}"] = np.array([np.linalg.norm(x)])
        out[f"pnorm_{tag}"] = np.array([np.sqrt(np.sum(dv ** 2))])
    del xa, xg
    j, _ = ref.sample_gaussian(ref.substream(GRAD_ROOT, 0, 0), 0, D, D)
    mid = ref.apply_lowrank_damped_inverse(ua, da, LAM, j, "right")
    del j
    s = ref.apply_lowrank_damped_inverse(ug, dg, LAM, mid, "left")
    del mid
    print(f"apply done at {time.time() - t0:.0f}s", flush=True)
    out["sv"] = (s @ v).astype(np.float32)
    out["ws"] = (w.T @ s).astype(np.float32)
    out["snorm"] = np.array([np.linalg.norm(s)])
    out["generator"] = np.array([f"oracle/_ref ({ref.kind}); {time.time() - t0:.0f}s"])
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, flush=True)


if __name__ == "__main__":
    main()
