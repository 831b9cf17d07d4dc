"""Seeded synthetic inputs for the SSE hot path (contract: include/qt_gen.h).

Holds no SSE arithmetic. Host fills (numpy) feed the oracle; device fills
(torch CUDA tensors) feed the product path; tests check both agree bit-for-bit.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .geometry import CONFIGS, neighbor_table, random_graph, reverse_slots  # noqa: F401

_HERE = Path(__file__).resolve().parent
SEED = 191210024
RANDOM, INTEGER, DELTA, ZERO, PHYSICAL = 0, 1, 2, 3, 4
ID_DH, ID_GL, ID_GG, ID_DL, ID_DG = 1, 2, 3, 4, 5

_i64, _u64, _int, _vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
_host = None
_dev = None


def _load_host():
    global _host
    if _host is None:
        lib = ctypes.CDLL(str(_HERE / "libqtgen_host.so"))
        lib.qtgen_host_G.argtypes = [_u64, _int, _int] + [_i64] * 8 + [_vp]
        lib.qtgen_host_D.argtypes = [_u64, _int, _int] + [_i64] * 4 + [_vp, _i64, _i64, _i64, _vp]
        lib.qtgen_host_dH.argtypes = [_u64, _int, _int] + [_i64] * 3 + [_vp, _vp]
        _host = lib
    return _host


def _load_dev():
    global _dev
    if _dev is None:
        lib = ctypes.CDLL(str(_HERE / "libqtgen_dev.so"))
        lib.qtgen_dev_G.argtypes = [_u64, _int, _int] + [_i64] * 8 + [_vp, _vp]
        lib.qtgen_dev_D.argtypes = [_u64, _int, _int] + [_i64] * 4 + [_vp, _i64, _i64, _i64, _vp, _vp]
        lib.qtgen_dev_dH.argtypes = [_u64, _int, _int] + [_i64] * 3 + [_vp, _vp, _vp]
        for f in (lib.qtgen_dev_G, lib.qtgen_dev_D, lib.qtgen_dev_dH):
            f.restype = _int
        _dev = lib
    return _dev


@dataclass
class Problem:
    """Dimensions (paper symbols) + neighbour graph."""
    nbr: np.ndarray                # int32 [Na][Nb], -1 = empty slot
    Norb: int
    NE: int
    Nw: int
    Nkz: int
    Nqz: int = -1
    shift0: int = 1
    shift_step: int = 1
    name: str = "custom"
    extra: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.Nqz < 0:
            self.Nqz = self.Nkz
        self.nbr = np.ascontiguousarray(self.nbr, dtype=np.int32)

    @property
    def Na(self) -> int:
        return self.nbr.shape[0]

    @property
    def Nb(self) -> int:
        return self.nbr.shape[1]

    @property
    def npairs(self) -> int:
        return int((self.nbr >= 0).sum())

    def shapes(self):
        return dict(G=(self.Nkz, self.NE, self.Na, self.Norb, self.Norb),
                    D=(self.Nqz, self.Nw, self.Na, self.Nb + 1, 3, 3),
                    dH=(self.Na, self.Nb, 3, self.Norb, self.Norb))


def problem(name: str) -> Problem:
    c = CONFIGS[name]
    return Problem(neighbor_table(*c["cells"], c["Nb"]), c["Norb"], c["NE"], c["Nw"], c["Nkz"], name=name)


# ---------------------------------------------------------------- host fills
def host_G(p: Problem, tid: int, mode: int = RANDOM, seed: int = SEED, e_lo=0, e_hi=None, a_lo=0, a_hi=None):
    e_hi = p.NE if e_hi is None else e_hi
    a_hi = p.Na if a_hi is None else a_hi
    out = np.empty((p.Nkz, e_hi - e_lo, a_hi - a_lo, p.Norb, p.Norb), dtype=np.complex128)
    _load_host().qtgen_host_G(seed, tid, mode, p.Nkz, p.NE, p.Na, p.Norb, e_lo, e_hi, a_lo, a_hi,
                              out.ctypes.data)
    return out


def host_D(p: Problem, tid: int, mode: int = RANDOM, seed: int = SEED, delta_m: int = 0, a_lo=0, a_hi=None):
    a_hi = p.Na if a_hi is None else a_hi
    out = np.empty((p.Nqz, p.Nw, a_hi - a_lo, p.Nb + 1, 3, 3), dtype=np.complex128)
    _load_host().qtgen_host_D(seed, tid, mode, p.Nqz, p.Nw, p.Na, p.Nb, p.nbr.ctypes.data, delta_m, a_lo, a_hi,
                              out.ctypes.data)
    return out


def host_dH(p: Problem, mode: int = RANDOM, seed: int = SEED):
    out = np.empty((p.Na, p.Nb, 3, p.Norb, p.Norb), dtype=np.complex128)
    _load_host().qtgen_host_dH(seed, ID_DH, mode, p.Na, p.Nb, p.Norb, p.nbr.ctypes.data, out.ctypes.data)
    return out


def host_inputs(p: Problem, mode: int = RANDOM, seed: int = SEED, dmode: int | None = None, delta_m: int = 0):
    """dict of host inputs. dmode overrides the D mode (DELTA puts δ in D^< only, D^> = 0)."""
    dm = mode if dmode is None else dmode
    return dict(
        dH=host_dH(p, mode, seed),
        G_less=host_G(p, ID_GL, mode, seed),
        G_gtr=host_G(p, ID_GG, mode, seed),
        D_less=host_D(p, ID_DL, dm, seed, delta_m),
        D_gtr=host_D(p, ID_DG, ZERO if dm == DELTA else dm, seed, delta_m),
    )


# ---------------------------------------------------------------- device fills (torch)
def _stream_ptr(stream):
    return None if stream is None else stream.cuda_stream


def dev_G(p: Problem, tid: int, out, mode: int = RANDOM, seed: int = SEED, e_lo=0, e_hi=None, a_lo=0, a_hi=None,
          stream=None):
    e_hi = p.NE if e_hi is None else e_hi
    a_hi = p.Na if a_hi is None else a_hi
    rc = _load_dev().qtgen_dev_G(seed, tid, mode, p.Nkz, p.NE, p.Na, p.Norb, e_lo, e_hi, a_lo, a_hi,
                                 out.data_ptr(), _stream_ptr(stream))
    if rc:
        raise RuntimeError(f"qtgen_dev_G failed: cuda error {rc}")


def dev_D(p: Problem, tid: int, out, nbr_dev, mode: int = RANDOM, seed: int = SEED, delta_m: int = 0, a_lo=0,
          a_hi=None, stream=None):
    a_hi = p.Na if a_hi is None else a_hi
    rc = _load_dev().qtgen_dev_D(seed, tid, mode, p.Nqz, p.Nw, p.Na, p.Nb, nbr_dev.data_ptr(), delta_m, a_lo, a_hi,
                                 out.data_ptr(), _stream_ptr(stream))
    if rc:
        raise RuntimeError(f"qtgen_dev_D failed: cuda error {rc}")


def dev_dH(p: Problem, out, nbr_dev, mode: int = RANDOM, seed: int = SEED, stream=None):
    rc = _load_dev().qtgen_dev_dH(seed, ID_DH, mode, p.Na, p.Nb, p.Norb, nbr_dev.data_ptr(), out.data_ptr(),
                                  _stream_ptr(stream))
    if rc:
        raise RuntimeError(f"qtgen_dev_dH failed: cuda error {rc}")


def dev_inputs(p: Problem, mode: int = RANDOM, seed: int = SEED, dmode: int | None = None, delta_m: int = 0,
               device="cuda"):
    import torch
    dm = mode if dmode is None else dmode
    sh = p.shapes()
    nbr_dev = torch.from_numpy(p.nbr).to(device)
    t = dict(dH=torch.empty(sh["dH"], dtype=torch.complex128, device=device),
             G_less=torch.empty(sh["G"], dtype=torch.complex128, device=device),
             G_gtr=torch.empty(sh["G"], dtype=torch.complex128, device=device),
             D_less=torch.empty(sh["D"], dtype=torch.complex128, device=device),
             D_gtr=torch.empty(sh["D"], dtype=torch.complex128, device=device))
    dev_dH(p, t["dH"], nbr_dev, mode, seed)
    dev_G(p, ID_GL, t["G_less"], mode, seed)
    dev_G(p, ID_GG, t["G_gtr"], mode, seed)
    dev_D(p, ID_DL, t["D_less"], nbr_dev, dm, seed, delta_m)
    dev_D(p, ID_DG, t["D_gtr"], nbr_dev, ZERO if dm == DELTA else dm, seed, delta_m)
    return t
