"""The hand-written d x d eigensolver (csrc/symeig.cu) of the exact K-FAC comparator and the
spectrum snapshots (8(f) #4), against eig.hpp:210-237 sym_eig through the oracle on the same (FP32-valued) inputs;
numpy's LAPACK eigh is the FP64 checker where the scalar oracle would take minutes (d >= 2305).

Bars: the solver computes in FP64 and returns FP32 eigenvectors, FP32 or FP64 eigenvalues.  Eigenvalues (FP64 out)
within 1e-10 * max|lambda| of the oracle's; reconstruction |P D P^T - S|_F / |S|_F <= 1e-6 and orthogonality
|P^T P - I|_max <= 1e-6 (FP32 storage of P).  Clusters (rank-deficient EA factors: thousands of zero eigenvalues,
a repeated spectrum) exercise the divide-and-conquer deflation."""
import numpy as np
import pytest

from tests.helpers import build_factor, psd_with_spectrum

pytestmark = pytest.mark.gpu


def t32(a, dev):
    import torch

    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32), device=dev)


def _check(rk, cuda, x32, d_ref, what):
    import torch

    s = t32(x32, cuda)
    res = rk.sym_eig(s)
    d64 = rk.sym_eigvals(s).cpu().numpy()
    torch.cuda.synchronize()
    p = res.p.double().cpu().numpy()
    dv = res.d.double().cpu().numpy()
    x = np.asarray(x32, np.float64)
    scale = max(np.abs(d_ref).max(), 1e-300)
    e_eig = np.abs(d64 - d_ref).max() / scale
    e_rec = np.linalg.norm((p * dv) @ p.T - x) / max(np.linalg.norm(x), 1e-300)
    e_orth = np.abs(p.T @ p - np.eye(x.shape[0])).max()
    print(f"{what}: eig {e_eig:.2e}, recon {e_rec:.2e}, orth {e_orth:.2e}")
    assert np.all(np.diff(d64) <= 0.0), "eigenvalues must be descending (eig.hpp:197-203)"
    assert e_eig <= 1e-10, (what, e_eig)
    assert e_rec <= 1e-6 and e_orth <= 1e-6, (what, e_rec, e_orth)


@pytest.mark.parametrize("d,steps", [(65, 3), (384, 6), (1153, 20)])
def test_sym_eig_matches_oracle_on_ea_factors(port, cuda, d, steps):
    import paper_2206_15397_b200 as rk

    x = build_factor(port, d, 128, steps, 1.0, f=0).astype(np.float32).astype(np.float64)
    _, d0 = port.sym_eig(x)
    _check(rk, cuda, x, d0, f"EA factor d={d}")


def test_sym_eig_rank_deficient_cluster(port, cuda):
    """One EA step from zero: rank 128 of 1153, ~1025 eigenvalues at 0 (one huge deflated cluster)."""
    import paper_2206_15397_b200 as rk

    x = build_factor(port, 1153, 128, 1, 1.0, f=0).astype(np.float32).astype(np.float64)
    _, d0 = port.sym_eig(x)
    _check(rk, cuda, x, d0, "rank 128 of 1153")


def test_sym_eig_repeated_and_small_sizes(port, cuda):
    import paper_2206_15397_b200 as rk

    eigs = np.repeat([5.0, 2.0, 2.0, 1e-3, 0.0], 40)  # 200 x 200 with four multiplicity-40/80 clusters
    x = psd_with_spectrum(port, eigs, 17).astype(np.float32).astype(np.float64)
    _, d0 = port.sym_eig(x)
    _check(rk, cuda, x, d0, "repeated spectrum")
    for n in (1, 2, 3, 31, 32, 33, 64):
        g, _ = port.sample_gaussian(100 + n, 0, n, n)
        x = (0.5 * (g + g.T)).astype(np.float32).astype(np.float64)  # indefinite
        _, d0 = port.sym_eig(x)
        _check(rk, cuda, x, d0, f"gaussian n={n}")


@pytest.mark.parametrize("d", [2305, 4609])
def test_sym_eig_vgg_sizes_vs_lapack(port, cuda, d):
    import paper_2206_15397_b200 as rk

    x = build_factor(port, d, 128, 4, 1.0, f=0).astype(np.float32).astype(np.float64)
    d0 = np.linalg.eigvalsh(x)[::-1]
    _check(rk, cuda, x, d0, f"EA factor d={d}")


def test_sym_eig_rejects_asymmetry(cuda):
    import torch
    import paper_2206_15397_b200 as rk

    s = torch.eye(4, device=cuda)
    s[0, 1] = 1.0
    with pytest.raises(rk.DimensionMismatch):
        rk.sym_eig(s)
