"""Seeded synthetic inputs for the RGF solver (include/qt_rgf.h): block-tridiagonal A = E·I − H − Σ^R with
Hermitian H (random Hermitian diagonal blocks, random couplings), anti-Hermitian block-diagonal Σ^≷, and the
retarded part Σ^R = (Σ^> − Σ^<)/2 (so that Σ^> − Σ^< = Σ^R − Σ^A, the convention of SPEC S:258). Holds no RGF
arithmetic (no inversion, no products of A blocks): only the problem setup of Eq. 1.

Host (numpy) fills feed the oracle and the small parity tests; device (torch CUDA) fills the bench-size runs.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEED = 191210024


@dataclass
class RgfProblem:
    P: int       # points (energies of one kz)
    bnum: int    # diagonal blocks
    bs: int      # block size (Na·Norb / bnum)
    name: str = "custom"

    @property
    def N(self) -> int:
        return self.bnum * self.bs


# test / bench shapes. rgf_finfet: the cfg3 FinFET slice (4,864 atoms, Norb = 10) cut into bnum = 76 blocks of 64
# atoms (bs = 640), 16 energy points.
CONFIGS = {
    "rgf_tiny": dict(P=3, bnum=4, bs=8),
    "rgf_small": dict(P=8, bnum=8, bs=48),
    "rgf_mid": dict(P=4, bnum=6, bs=160),
    "rgf_finfet": dict(P=16, bnum=76, bs=640),
}


def problem(name: str) -> RgfProblem:
    return RgfProblem(name=name, **CONFIGS[name])


def energies(p: RgfProblem):
    return np.linspace(-1.0, 1.0, p.P)


def host_inputs(p: RgfProblem, seed: int = SEED, eta: float = 1e-3, coupling: float = 0.5, scatter: float = 0.2):
    """dict of complex128 numpy arrays Ad [P][bnum][bs][bs], Au/Al [P][bnum-1][bs][bs], Sl/Sg [P][bnum][bs][bs]."""
    rng = np.random.default_rng(seed)
    P, nb, bs = p.P, p.bnum, p.bs

    def cplx(*shape):
        return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)

    Hd = cplx(nb, bs, bs) / np.sqrt(bs)
    Hd = (Hd + np.conj(np.swapaxes(Hd, -1, -2))) / 2
    Hu = coupling * cplx(max(nb - 1, 0), bs, bs) / np.sqrt(bs)
    X = cplx(P, nb, bs, bs) / np.sqrt(bs)
    Y = cplx(P, nb, bs, bs) / np.sqrt(bs)
    Sl = 1j * scatter * (X @ np.conj(np.swapaxes(X, -1, -2)))
    Sg = -1j * scatter * (Y @ np.conj(np.swapaxes(Y, -1, -2)))
    SR = (Sg - Sl) / 2
    E = energies(p)
    eye = np.eye(bs)
    Ad = (E[:, None, None, None] + 1j * eta) * eye - Hd[None] - SR
    Au = np.broadcast_to(-Hu[None], (P, max(nb - 1, 0), bs, bs)).copy()
    Al = np.broadcast_to(-np.conj(np.swapaxes(Hu, -1, -2))[None], (P, max(nb - 1, 0), bs, bs)).copy()
    return dict(Ad=np.ascontiguousarray(Ad), Au=Au, Al=Al, Sl=np.ascontiguousarray(Sl), Sg=np.ascontiguousarray(Sg))


def dev_inputs(p: RgfProblem, seed: int = SEED, eta: float = 1e-3, coupling: float = 0.5, scatter: float = 0.2,
               device="cuda"):
    """Same construction on the device with torch's CUDA generator (bench sizes; not bit-identical to host)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    P, nb, bs = p.P, p.bnum, p.bs
    c128 = torch.complex128

    def cplx(*shape):
        return torch.randn(shape, dtype=c128, device=device, generator=g) * np.sqrt(2.0)   # re, im ~ N(0, 1)

    Hd = cplx(nb, bs, bs) / np.sqrt(bs)
    Hd = (Hd + Hd.transpose(-1, -2).conj()) / 2
    Hu = coupling * cplx(max(nb - 1, 0), bs, bs) / np.sqrt(bs)
    E = torch.tensor(energies(p), dtype=torch.float64, device=device)
    eye = torch.eye(bs, dtype=c128, device=device)
    out = dict(Ad=torch.empty((P, nb, bs, bs), dtype=c128, device=device),
               Sl=torch.empty((P, nb, bs, bs), dtype=c128, device=device),
               Sg=torch.empty((P, nb, bs, bs), dtype=c128, device=device))
    for q in range(P):   # one point at a time: bounded temporaries
        X = cplx(nb, bs, bs) / np.sqrt(bs)
        out["Sl"][q] = 1j * scatter * (X @ X.transpose(-1, -2).conj())
        X = cplx(nb, bs, bs) / np.sqrt(bs)
        out["Sg"][q] = -1j * scatter * (X @ X.transpose(-1, -2).conj())
        out["Ad"][q] = (E[q] + 1j * eta) * eye - Hd - (out["Sg"][q] - out["Sl"][q]) / 2
    out["Au"] = (-Hu).unsqueeze(0).expand(P, -1, -1, -1).contiguous()
    out["Al"] = (-Hu.transpose(-1, -2).conj()).unsqueeze(0).expand(P, -1, -1, -1).contiguous()
    return out
