"""Gram matrix, SVD and symmetric eigendecomposition on the GPU (SURVEY.md
§8f item 3: "Gram Λ^ν and SVD on device for large M").

The reference does these on the host in float64 (S/estimator.py:112-118
``_gram``; S/linalg.py ``svd`` / ``sym_eig``, used by S/tsvd.py:48-130;
S/ = /root/reference/pkg/src/exitmeasure/).  At cfg5's size (4096 poles x
4096 Γ1 cells) the host Gram is a 1.4e11-flop DGEMM and the SVD/eigh take
seconds; here they run in float64 on the B200 (cuBLAS DGEMM, cuSOLVER
SVD / syevd through torch -- plain library calls, the walk kernel is the
hand-written part).  ``gram_from_counts`` starts from the int64 count rows a
``Plan.run_device`` left in HBM, so the estimator never round-trips A through
the host.

Results agree with the host routines to float64 rounding (the summation
order differs), not bit for bit; singular/eigen vectors are unique up to
sign (and rotation inside exactly degenerate subspaces), which the
reconstructions built from them (S/tsvd.py:93-130) do not see.  There is no
CPU fallback: without a CUDA device these raise NativeError.
"""

from __future__ import annotations

import numpy as np

from .errors import NativeError, ValidationError


def _torch_device(device: int | None):
    import torch

    if not torch.cuda.is_available():
        raise NativeError("spectral routines run on the GPU only (no CUDA device visible)")
    return torch.device("cuda", 0 if device is None else int(device))


def _require_matrix(a, name: str) -> np.ndarray:
    """Mirror of S/linalg.py:51-57 (2-D, finite)."""
    a = np.asarray(a, dtype=float)
    if a.ndim != 2:
        raise ValidationError(f"{name} must be a matrix, got ndim={a.ndim}")
    if not np.all(np.isfinite(a)):
        raise ValidationError(f"{name} has non-finite entries")
    return a


def _mirror_upper(g):
    """Copy the strict upper triangle onto the lower one, as the reference
    does so the stored Gram is exactly symmetric (S/estimator.py:115-117)."""
    import torch

    return torch.triu(g) + torch.triu(g, diagonal=1).transpose(0, 1)


def gram_device(a1, sigma1, nu, device: int | None = None):
    """Λ^ν = M M^T, M = diag(ν) A1 diag(σ)^{-1/2}, as a float64 CUDA tensor.
    ``a1`` may be a host array or a CUDA tensor (poles x Γ1 cells)."""
    import torch

    dev = _torch_device(device)
    a = torch.as_tensor(a1, dtype=torch.float64, device=dev)
    s = torch.as_tensor(np.asarray(sigma1, dtype=float), device=dev)
    v = torch.as_tensor(np.asarray(nu, dtype=float), device=dev)
    if a.ndim != 2 or s.shape[0] != a.shape[1] or v.shape[0] != a.shape[0]:
        raise ValidationError("gram: a1 (M, M1), sigma1 (M1,), nu (M,) required")
    m = (v[:, None] * a) / torch.sqrt(s)[None, :]
    return _mirror_upper(m @ m.transpose(0, 1))


def gram(a1, sigma1, nu, device: int | None = None) -> np.ndarray:
    """Drop-in for S/estimator.py:112-118 ``_gram`` (host arrays in and out)."""
    return gram_device(a1, sigma1, nu, device).cpu().numpy()


def gram_from_counts(counts, n0: int, n_rep: int, sigma1, nu, device: int | None = None):
    """Λ^ν straight from a run's int64 count rows on the device: A1 =
    counts[:, n0:] / n_rep (the reference's ``res.raw1 / n``,
    S/estimator.py:150), never copied to the host."""
    import torch

    c = counts if isinstance(counts, torch.Tensor) else torch.as_tensor(counts)
    dev = _torch_device(device if device is not None else
                        (c.device.index if c.is_cuda else None))
    a1 = c.to(dev)[:, int(n0):].to(torch.float64) / float(n_rep)
    return gram_device(a1, sigma1, nu, dev.index)


def svd(b, device: int | None = None):
    """Full SVD factors (U, s, V), B = U diag(s) V^T, s descending: drop-in for
    S/linalg.py ``svd`` (full_matrices=True)."""
    import torch

    b = _require_matrix(b, "B")
    dev = _torch_device(device)
    u, s, vh = torch.linalg.svd(torch.as_tensor(b, device=dev), full_matrices=True)
    return u.cpu().numpy(), s.cpu().numpy(), vh.transpose(0, 1).cpu().numpy()


def sym_eig(a, device: int | None = None):
    """Eigenvalues (descending) and orthonormal eigenvector columns of a
    symmetric matrix: drop-in for S/linalg.py ``sym_eig`` (same square and
    1e-12 relative symmetry checks)."""
    import torch

    a = _require_matrix(a, "A")
    n, m = a.shape
    if n != m:
        raise ValidationError(f"A must be square, got {n}x{m}")
    scale = np.max(np.abs(a)) if a.size else 0.0
    scale = scale or 1.0
    if np.max(np.abs(a - a.T)) > 1e-12 * scale:
        raise ValidationError("A is not symmetric to 1e-12 relative")
    dev = _torch_device(device)
    w, v = torch.linalg.eigh(torch.as_tensor(a, device=dev))
    return w.flip(0).cpu().numpy(), v.flip(1).cpu().numpy()
