"""CPU oracle of the RGF workload — TEST INFRASTRUCTURE ONLY (same rule as oracle/__init__.py).

The plain definition of Eq. 1: assemble the full block-tridiagonal A of each point, invert it
densely (numpy.linalg.inv, a library primitive used as one step), and form G^≷ = G^R Σ^≷ G^A with dense
products; return the diagonal blocks. No recursion, no blocking: the RGF pass is what the GPU path
does and what this checks. Pinned in tests/test_rgf_oracle.py (residual A·G^R = I, the Σ^> − Σ^< = Σ^R − Σ^A ⇒
G^> − G^< = G^R − G^A identity, anti-Hermiticity, the identity-matrix example of SPEC S:229, and the two-site
closed form).
"""
from __future__ import annotations

import numpy as np


def assemble(Ad, Au, Al, p):
    """Full A [N][N] of point p from its blocks."""
    nb, bs = Ad.shape[1], Ad.shape[2]
    A = np.zeros((nb * bs, nb * bs), dtype=np.complex128)
    for n in range(nb):
        A[n * bs:(n + 1) * bs, n * bs:(n + 1) * bs] = Ad[p, n]
        if n + 1 < nb:
            A[n * bs:(n + 1) * bs, (n + 1) * bs:(n + 2) * bs] = Au[p, n]
            A[(n + 1) * bs:(n + 2) * bs, n * bs:(n + 1) * bs] = Al[p, n]
    return A


def block_diag(S, p):
    nb, bs = S.shape[1], S.shape[2]
    M = np.zeros((nb * bs, nb * bs), dtype=np.complex128)
    for n in range(nb):
        M[n * bs:(n + 1) * bs, n * bs:(n + 1) * bs] = S[p, n]
    return M


def diag_blocks(M, nb, bs):
    return np.stack([M[n * bs:(n + 1) * bs, n * bs:(n + 1) * bs] for n in range(nb)])


def solve(inp, points=None):
    """Diagonal blocks of G^R, G^<, G^> [P'][bnum][bs][bs] for the given points (default: all)."""
    Ad, Au, Al, Sl, Sg = (inp[k] for k in ("Ad", "Au", "Al", "Sl", "Sg"))
    P, nb, bs = Ad.shape[0], Ad.shape[1], Ad.shape[2]
    pts = range(P) if points is None else points
    GR, GL, GG = [], [], []
    for p in pts:
        A = assemble(Ad, Au, Al, p)
        R = np.linalg.inv(A)                      # G^R = A^{-1}
        Ra = np.conj(R.T)                         # G^A = (G^R)†
        GR.append(diag_blocks(R, nb, bs))
        GL.append(diag_blocks(R @ block_diag(Sl, p) @ Ra, nb, bs))   # G^< = G^R Σ^< G^A
        GG.append(diag_blocks(R @ block_diag(Sg, p) @ Ra, nb, bs))   # G^> = G^R Σ^> G^A
    return np.stack(GR), np.stack(GL), np.stack(GG)
