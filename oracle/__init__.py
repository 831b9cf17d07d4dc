"""CPU oracle for Σ≷ (Eq. 3) and Π≷ (Eq. 4) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package. The product path never does.

Functions follow PAPER.md Eq. 3 and Eq. 4 with the
readings R1-R19 listed in DESIGN.md §3 (see oracle/oracle.c for the loops).
`brute_*` is an independent scalarized six-loop evaluation for
tiny inputs, used to pin the oracle (pin P1).
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_lib = None


class _Dims(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("Na", "Nb", "Norb", "NE", "Nw", "Nkz", "Nqz", "shift0", "shift_step")]


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(str(_HERE / "liboracle.so"))
        P, D, I = ctypes.c_void_p, ctypes.c_double, ctypes.c_int64
        lib.oracle_sigma.argtypes = [P, P, P, P, P, P, P, D, D, P, P]
        lib.oracle_pi.argtypes = [P, P, P, P, P, D, D, P, P]
        lib.oracle_sigma_blocks.argtypes = [P, P, P, P, P, P, P, D, D, I, P, P]
        lib.oracle_pi_blocks.argtypes = [P, P, P, P, P, D, D, I, P, P]
        lib.brute_sigma.argtypes = [P, P, P, P, P, P, P, D, D, P, P]
        lib.brute_pi.argtypes = [P, P, P, P, P, D, D, P, P]
        _lib = lib
    return _lib


def set_threads(n: int | None) -> None:
    """OpenMP thread count for subsequent oracle calls (None = leave the default)."""
    if n is not None:
        os.environ["OMP_NUM_THREADS"] = str(n)


def _dims(p):
    return _Dims(p.Na, p.Nb, p.Norb, p.NE, p.Nw, p.Nkz, p.Nqz, p.shift0, p.shift_step)


def _c(x):
    return np.ascontiguousarray(x, dtype=np.complex128)


def sigma(p, inp, scale=1j):
    """Full Σ^<, Σ^> [Nkz][NE][Na][Norb][Norb] (Eq. 3)."""
    lib = _load()
    d = _dims(p)
    ins = [_c(inp[k]) for k in ("dH", "G_less", "G_gtr", "D_less", "D_gtr")]
    SL = np.zeros(p.shapes()["G"], dtype=np.complex128)
    SG = np.zeros_like(SL)
    lib.oracle_sigma(ctypes.byref(d), p.nbr.ctypes.data, *[a.ctypes.data for a in ins], scale.real, scale.imag,
                     SL.ctypes.data, SG.ctypes.data)
    return SL, SG


def pi(p, inp, scale=-1j):
    """Full Π^<, Π^> [Nqz][Nw][Na][Nb+1][3][3] (Eq. 4)."""
    lib = _load()
    d = _dims(p)
    ins = [_c(inp[k]) for k in ("dH", "G_less", "G_gtr")]
    PL = np.zeros(p.shapes()["D"], dtype=np.complex128)
    PG = np.zeros_like(PL)
    lib.oracle_pi(ctypes.byref(d), p.nbr.ctypes.data, *[a.ctypes.data for a in ins], scale.real, scale.imag,
                  PL.ctypes.data, PG.ctypes.data)
    return PL, PG


def sigma_blocks(p, inp, blocks, scale=1j):
    """Σ blocks for rows (X, kz, e, a) of `blocks` (X: 0 '<', 1 '>'). -> [n][Norb][Norb]."""
    lib = _load()
    d = _dims(p)
    blk = np.ascontiguousarray(blocks, dtype=np.int64).reshape(-1, 4)
    ins = [_c(inp[k]) for k in ("dH", "G_less", "G_gtr", "D_less", "D_gtr")]
    out = np.zeros((blk.shape[0], p.Norb, p.Norb), dtype=np.complex128)
    lib.oracle_sigma_blocks(ctypes.byref(d), p.nbr.ctypes.data, *[a.ctypes.data for a in ins], scale.real,
                            scale.imag, blk.shape[0], blk.ctypes.data, out.ctypes.data)
    return out


def pi_blocks(p, inp, blocks, scale=-1j):
    """Π blocks for rows (X, qz, m, a, slot) of `blocks`. -> [n][3][3]."""
    lib = _load()
    d = _dims(p)
    blk = np.ascontiguousarray(blocks, dtype=np.int64).reshape(-1, 5)
    ins = [_c(inp[k]) for k in ("dH", "G_less", "G_gtr")]
    out = np.zeros((blk.shape[0], 3, 3), dtype=np.complex128)
    lib.oracle_pi_blocks(ctypes.byref(d), p.nbr.ctypes.data, *[a.ctypes.data for a in ins], scale.real,
                         scale.imag, blk.shape[0], blk.ctypes.data, out.ctypes.data)
    return out


def brute_sigma(p, inp, scale=1j):
    lib = _load()
    d = _dims(p)
    ins = [_c(inp[k]) for k in ("dH", "G_less", "G_gtr", "D_less", "D_gtr")]
    SL = np.zeros(p.shapes()["G"], dtype=np.complex128)
    SG = np.zeros_like(SL)
    lib.brute_sigma(ctypes.byref(d), p.nbr.ctypes.data, *[a.ctypes.data for a in ins], scale.real, scale.imag,
                    SL.ctypes.data, SG.ctypes.data)
    return SL, SG


def brute_pi(p, inp, scale=-1j):
    lib = _load()
    d = _dims(p)
    ins = [_c(inp[k]) for k in ("dH", "G_less", "G_gtr")]
    PL = np.zeros(p.shapes()["D"], dtype=np.complex128)
    PG = np.zeros_like(PL)
    lib.brute_pi(ctypes.byref(d), p.nbr.ctypes.data, *[a.ctypes.data for a in ins], scale.real, scale.imag,
                 PL.ctypes.data, PG.ctypes.data)
    return PL, PG


# ---------------------------------------------------------------- paper flop model (reporting)
def paper_flops_omen(Na, Nb, N3D, Nkz, Nqz, NE, Nw, Norb):
    """OMEN SSE flop count, §5.1.1: 64·Na·Nb·N3D·Nkz·Nqz·NE·Nω·Norb³."""
    return 64.0 * Na * Nb * N3D * Nkz * Nqz * NE * Nw * Norb ** 3


def paper_flops_dace(Na, Nb, N3D, Nkz, Nqz, NE, Nw, Norb, plus=1):
    """DaCe SSE flops: OMEN ÷ 2NqzNω/(NqzNω+1). `plus`=N3D fits Table 2 (reading R15)."""
    return paper_flops_omen(Na, Nb, N3D, Nkz, Nqz, NE, Nw, Norb) * (Nqz * Nw + plus) / (2.0 * Nqz * Nw)
