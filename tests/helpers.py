"""Shared parity metrics and input builders (test infrastructure; uses the CPU oracle as the checker)."""
from __future__ import annotations

import numpy as np

ROOT_SEED = 220615397  # synthetic factor statistics
OMEGA_ROOT = 7         # Omega substream root
GRAD_ROOT = 99         # gradient substream root


def build_factor(port, d: int, n: int, steps: int, e: float, f: int = 0, rho: float = 0.95, zero_init=True):
    """EA factor from `steps` synthetic updates, FP64, via the oracle."""
    x = np.zeros((d, d)) if zero_init else np.eye(d)
    for k in range(steps):
        m = port.synthetic_m(ROOT_SEED, k, f, n, d, e)
        x = port.ea_update(x, m, rho)
    return x


def recon(u, dv):
    u = np.asarray(u, np.float64)
    return (u * np.asarray(dv, np.float64)[None, :]) @ u.T


def recon_err(u1, d1, u0, d0) -> float:
    a, b = recon(u1, d1), recon(u0, d0)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def eig_err(d1, d0, floor: float = 0.0) -> float:
    d1 = np.asarray(d1, np.float64); d0 = np.asarray(d0, np.float64)
    den = np.maximum(np.abs(d0), floor)
    den = np.where(den > 0, den, 1.0)
    return float(np.max(np.abs(d1 - d0) / den)) if d0.size else 0.0


def rel_fro(a, b) -> float:
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def orth_err(u) -> float:
    u = np.asarray(u, np.float64)
    return float(np.max(np.abs(u.T @ u - np.eye(u.shape[1])))) if u.size else 0.0


def psd_with_spectrum(port, eigs, seed):
    """test_util.hpp:107-116 through the oracle (qr_thin of a seeded Gaussian)."""
    n = len(eigs)
    g, _ = port.sample_gaussian(seed, 0, n, n)
    q, _ = port.qr_thin(g)
    x = (q * np.asarray(eigs)[None, :]) @ q.T
    return 0.5 * (x + x.T)


def geometric_spectrum(n, ratio=0.9):
    return ratio ** np.arange(n, dtype=np.float64)
