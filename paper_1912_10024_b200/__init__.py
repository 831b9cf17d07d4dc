"""B200-native electron-phonon scattering self-energy (SSE) hot path of
Ziogas et al., SC19 (arXiv 1912.10024): Σ≷ (Eq. 3) and Π≷ (Eq. 4).

Thin ctypes binding over the C ABI of libqtsse.so (include/qt_sse.h): argument
marshalling only — every step of the path runs in the library's sm_100a kernels.
There is no CPU fallback: importing fails loudly when the library is missing.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libqtsse.so"

QT_OK, QT_ERR_INVALID_ARG, QT_ERR_UNSUPPORTED, QT_ERR_OUT_OF_MEMORY, QT_ERR_CUDA, QT_ERR_NCCL, QT_ERR_INTERNAL = range(7)
QT_SHARD_NONE, QT_SHARD_ENERGY, QT_SHARD_ATOM, QT_SHARD_2D = range(4)
QT_FLAG_DETERMINISTIC = 1
QT_PREC_FP64, QT_PREC_FP32_MIXED = 0, 1
EXPORTED = ["qt_sse_plan", "qt_sse_sigma", "qt_sse_pi", "qt_sse_execute_host", "qt_sse_query",
            "qt_sse_halo_exchange", "qt_sse_destroy", "qt_sse_status_string", "qt_sse_count_flops",
            "qt_sse_launch_count", "qt_sse_timing_enable", "qt_sse_timing_read", "qt_sse_nccl_unique_id",
            "qt_sse_shard_info", "qt_sse_sigma_pi"]
EXPORTED_RGF = ["qt_rgf_plan", "qt_rgf_solve", "qt_rgf_check_info", "qt_rgf_count_flops", "qt_rgf_destroy"]
KERNEL_KINDS = ["k_sigma_coef", "k_sigma", "k_pi_w", "k_pi_contract", "k_pi_self", "k_relayout", "k_halo_pack",
                "k_sigma_sand", "k_sigma_pair"]


class Desc(ctypes.Structure):
    _fields_ = [("Na", ctypes.c_int64), ("Nb", ctypes.c_int64), ("Norb", ctypes.c_int64), ("N3D", ctypes.c_int64),
                ("NE", ctypes.c_int64), ("Nw", ctypes.c_int64), ("Nkz", ctypes.c_int64), ("Nqz", ctypes.c_int64),
                ("shift0", ctypes.c_int32), ("shift_step", ctypes.c_int32), ("precision", ctypes.c_int),
                ("shard", ctypes.c_int), ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p), ("workspace_limit", ctypes.c_size_t),
                ("grid_atoms", ctypes.c_int32), ("flags", ctypes.c_uint32)]


class Info(ctypes.Structure):
    _fields_ = [("a_lo", ctypes.c_int64), ("a_hi", ctypes.c_int64), ("w_lo", ctypes.c_int64),
                ("w_hi", ctypes.c_int64), ("npairs", ctypes.c_int64), ("workspace_bytes", ctypes.c_size_t),
                ("flops_sigma", ctypes.c_double), ("flops_pi", ctypes.c_double), ("halo_bytes", ctypes.c_double),
                ("e_lo", ctypes.c_int64), ("e_hi", ctypes.c_int64), ("ew_lo", ctypes.c_int64), ("ew_hi", ctypes.c_int64),
                ("pa_lo", ctypes.c_int64), ("pa_hi", ctypes.c_int64), ("Ta", ctypes.c_int32), ("TE", ctypes.c_int32),
                ("ta", ctypes.c_int32), ("te", ctypes.c_int32), ("reduce_bytes", ctypes.c_double),
                ("mem_bytes", ctypes.c_double), ("flops_sigma_pair", ctypes.c_double)]


class RgfDesc(ctypes.Structure):
    _fields_ = [("P", ctypes.c_int64), ("bnum", ctypes.c_int64), ("bs", ctypes.c_int64)]


class QTError(RuntimeError):
    pass


def _load():
    if not _LIB_PATH.exists():
        raise ImportError(f"{_LIB_PATH} is missing: build it with `python -m paper_1912_10024_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(_LIB_PATH))
    P, D, I = ctypes.c_void_p, ctypes.c_double, ctypes.c_int
    lib.qt_sse_plan.argtypes = [ctypes.POINTER(Desc), P, P, ctypes.POINTER(P)]
    lib.qt_sse_sigma.argtypes = [P, P, P, P, P, P, D, D, P, P, P]
    lib.qt_sse_pi.argtypes = [P, P, P, P, D, D, P, P, P]
    lib.qt_sse_sigma_pi.argtypes = [P, P, P, P, P, P, D, D, D, D, P, P, P, P, P]
    lib.qt_sse_execute_host.argtypes = [P, P, P, P, P, P, D, D, D, D, P, P, P, P, P]
    lib.qt_sse_query.argtypes = [P, ctypes.POINTER(Info)]
    lib.qt_sse_halo_exchange.argtypes = [P, P, P, P, P, P]
    lib.qt_sse_destroy.argtypes = [P]
    lib.qt_sse_destroy.restype = None
    lib.qt_sse_status_string.argtypes = [I]
    lib.qt_sse_status_string.restype = ctypes.c_char_p
    lib.qt_sse_count_flops.argtypes = [ctypes.POINTER(Desc), P, ctypes.POINTER(ctypes.c_double)]
    lib.qt_sse_launch_count.argtypes = []
    lib.qt_sse_launch_count.restype = ctypes.c_uint64
    lib.qt_sse_nccl_unique_id.argtypes = [P]
    lib.qt_sse_shard_info.argtypes = [ctypes.POINTER(Desc), P, ctypes.POINTER(Info)]
    lib.qt_sse_timing_enable.argtypes = [P, I]
    lib.qt_sse_timing_read.argtypes = [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
    lib.qt_rgf_plan.argtypes = [ctypes.POINTER(RgfDesc), P, ctypes.POINTER(P)]
    lib.qt_rgf_solve.argtypes = [P, P, P, P, P, P, P, P, P, P]
    lib.qt_rgf_check_info.argtypes = [P, P, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
    lib.qt_rgf_count_flops.argtypes = [ctypes.POINTER(RgfDesc), ctypes.POINTER(ctypes.c_double)]
    lib.qt_rgf_destroy.argtypes = [P]
    lib.qt_rgf_destroy.restype = None
    for f in ("qt_rgf_plan", "qt_rgf_solve", "qt_rgf_check_info", "qt_rgf_count_flops"):
        getattr(lib, f).restype = I
    for f in ("qt_sse_plan", "qt_sse_sigma", "qt_sse_pi", "qt_sse_sigma_pi", "qt_sse_execute_host", "qt_sse_query",
              "qt_sse_halo_exchange", "qt_sse_count_flops", "qt_sse_timing_enable", "qt_sse_timing_read",
              "qt_sse_nccl_unique_id", "qt_sse_shard_info"):
        getattr(lib, f).restype = I
    return lib


_lib = None


def _get_lib():
    """Load libqtsse.so on first use (so the in-tree build can run before it exists)."""
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def __getattr__(name):   # PEP 562: `paper_1912_10024_b200.lib` is the loaded C library
    if name == "lib":
        return _get_lib()
    raise AttributeError(name)


def _check(rc: int, what: str) -> None:
    if rc != QT_OK:
        raise QTError(f"{what}: {_get_lib().qt_sse_status_string(rc).decode()} (status {rc})")


def make_desc(p, rank=0, nranks=1, shard=QT_SHARD_NONE, workspace_limit=0, unique_id=None,
              precision=QT_PREC_FP64, grid_atoms=0, flags=0) -> Desc:
    """Desc from a qtgen.Problem-like object (Na, Nb, Norb, NE, Nw, Nkz, Nqz, shift0, shift_step)."""
    return Desc(p.Na, p.Nb, p.Norb, 3, p.NE, p.Nw, p.Nkz, p.Nqz, p.shift0, p.shift_step, precision, shard, rank,
                nranks, unique_id, workspace_limit, grid_atoms, flags)


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for a sharded plan (create on one rank, broadcast to the others)."""
    buf = ctypes.create_string_buffer(128)
    _check(_get_lib().qt_sse_nccl_unique_id(buf), "qt_sse_nccl_unique_id")
    return buf.raw


def count_flops(p, rank=0, nranks=1, shard=QT_SHARD_NONE, grid_atoms=0) -> dict:
    """Algorithmic flops (F_alg) of the whole problem, or of one rank's block."""
    d = make_desc(p, rank=rank, nranks=nranks, shard=shard if nranks > 1 else QT_SHARD_NONE, grid_atoms=grid_atoms)
    out = (ctypes.c_double * 4)()
    nbr = np.ascontiguousarray(p.nbr, dtype=np.int32)
    _check(_get_lib().qt_sse_count_flops(ctypes.byref(d), nbr.ctypes.data, out), "qt_sse_count_flops")
    return dict(sigma_contraction=out[0], sigma_sandwich=out[1], pi_sandwich=out[2], pi_contraction=out[3],
                total=sum(out))


def shard_info(p, rank: int, nranks: int, shard=None, grid_atoms=0, workspace_limit=0,
               precision=QT_PREC_FP64) -> dict:
    """Host-only: owned atoms [a_lo,a_hi) / energies [e_lo,e_hi), input windows [w_lo,w_hi) / [ew_lo,ew_hi),
    Π output atoms [pa_lo,pa_hi), grid (Ta, TE, ta, te), pairs, flops, halo and reduction bytes, and the
    per-rank device footprint mem_bytes (atom sharding unless shard says otherwise)."""
    if shard is None:
        shard = QT_SHARD_ATOM if nranks > 1 else QT_SHARD_NONE
    d = make_desc(p, rank=rank, nranks=nranks, shard=shard, grid_atoms=grid_atoms, workspace_limit=workspace_limit,
                  precision=precision)
    i = Info()
    nbr = np.ascontiguousarray(p.nbr, dtype=np.int32)
    _check(_get_lib().qt_sse_shard_info(ctypes.byref(d), nbr.ctypes.data, ctypes.byref(i)), "qt_sse_shard_info")
    return {k: getattr(i, k) for k, _ in Info._fields_}


def launch_count() -> int:
    return int(_get_lib().qt_sse_launch_count())


def _ptr(t):
    return t.data_ptr() if hasattr(t, "data_ptr") else t.ctypes.data


def _stream(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


class Plan:
    """Owns a qt_sse_plan_t (workspace, work lists) for one problem shape."""

    def __init__(self, p, stream=None, workspace_limit=0, rank=0, nranks=1, shard=QT_SHARD_NONE, unique_id=None,
                 precision=QT_PREC_FP64, grid_atoms=0, flags=0):
        self._uid = None if unique_id is None else ctypes.create_string_buffer(bytes(unique_id), 128)
        self.desc = make_desc(p, rank=rank, nranks=nranks, shard=shard, workspace_limit=workspace_limit,
                              unique_id=None if self._uid is None else ctypes.addressof(self._uid),
                              precision=precision, grid_atoms=grid_atoms, flags=flags)
        self._nbr = np.ascontiguousarray(p.nbr, dtype=np.int32)
        h = ctypes.c_void_p()
        _check(_get_lib().qt_sse_plan(ctypes.byref(self.desc), self._nbr.ctypes.data, _stream(stream), ctypes.byref(h)),
               "qt_sse_plan")
        self.h = h

    def info(self) -> dict:
        i = Info()
        _check(_get_lib().qt_sse_query(self.h, ctypes.byref(i)), "qt_sse_query")
        return {k: getattr(i, k) for k, _ in Info._fields_}

    def sigma(self, dH, G_less, G_gtr, D_less, D_gtr, S_less, S_gtr, scale=1j, stream=None):
        _check(_get_lib().qt_sse_sigma(self.h, _ptr(dH), _ptr(G_less), _ptr(G_gtr), _ptr(D_less), _ptr(D_gtr),
                                scale.real, scale.imag, _ptr(S_less), _ptr(S_gtr), _stream(stream)), "qt_sse_sigma")

    def pi(self, dH, G_less, G_gtr, P_less, P_gtr, scale=-1j, stream=None):
        _check(_get_lib().qt_sse_pi(self.h, _ptr(dH), _ptr(G_less), _ptr(G_gtr), scale.real, scale.imag, _ptr(P_less),
                             _ptr(P_gtr), _stream(stream)), "qt_sse_pi")

    def sigma_pi(self, dH, G_less, G_gtr, D_less, D_gtr, S_less, S_gtr, P_less, P_gtr, sig_scale=1j, pi_scale=-1j,
                 stream=None):
        """The whole hot path in one call: halo exchange (sharded plans with a communicator) overlapped with the
        interior work, Σ≷ and Π≷ (G/D window halos are filled in place)."""
        _check(_get_lib().qt_sse_sigma_pi(self.h, _ptr(dH), _ptr(G_less), _ptr(G_gtr), _ptr(D_less), _ptr(D_gtr),
                                          sig_scale.real, sig_scale.imag, pi_scale.real, pi_scale.imag, _ptr(S_less),
                                          _ptr(S_gtr), _ptr(P_less), _ptr(P_gtr), _stream(stream)), "qt_sse_sigma_pi")

    def execute_host(self, dH, G_less, G_gtr, D_less, D_gtr, S_less, S_gtr, P_less, P_gtr, sig_scale=1j,
                     pi_scale=-1j, stream=None):
        """End-to-end on host buffers (numpy / pinned torch CPU tensors)."""
        _check(_get_lib().qt_sse_execute_host(self.h, _ptr(dH), _ptr(G_less), _ptr(G_gtr), _ptr(D_less), _ptr(D_gtr),
                                       sig_scale.real, sig_scale.imag, pi_scale.real, pi_scale.imag, _ptr(S_less),
                                       _ptr(S_gtr), _ptr(P_less), _ptr(P_gtr), _stream(stream)),
               "qt_sse_execute_host")

    def halo_exchange(self, G_less, G_gtr, D_less, D_gtr, stream=None):
        """Fill the halo region of this rank's input windows from their owners (NCCL, in place)."""
        _check(_get_lib().qt_sse_halo_exchange(self.h, _ptr(G_less), _ptr(G_gtr), _ptr(D_less), _ptr(D_gtr),
                                               _stream(stream)), "qt_sse_halo_exchange")

    def timing(self, enable: bool = True):
        _check(_get_lib().qt_sse_timing_enable(self.h, int(enable)), "qt_sse_timing_enable")

    def timing_read(self) -> dict:
        """{kernel: (ms_total, launches)} since the last read (synchronizes the recorded events)."""
        ms = (ctypes.c_double * len(KERNEL_KINDS))()
        n = (ctypes.c_int64 * len(KERNEL_KINDS))()
        _check(_get_lib().qt_sse_timing_read(self.h, ms, n), "qt_sse_timing_read")
        return {k: (ms[i], n[i]) for i, k in enumerate(KERNEL_KINDS)}

    def close(self):
        if self.h:
            _get_lib().qt_sse_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run(p, t: dict, sig_scale=1j, pi_scale=-1j, plan: Plan | None = None, precision=QT_PREC_FP64, fused=False,
        workspace_limit=0, flags=0):
    """Σ≷, Π≷ for device inputs t (dict of complex128 CUDA tensors as made by qtgen.dev_inputs); separate
    qt_sse_sigma + qt_sse_pi calls, or the fused qt_sse_sigma_pi."""
    import torch
    own = plan is None
    plan = Plan(p, precision=precision, workspace_limit=workspace_limit, flags=flags) if own else plan
    sh = p.shapes()
    out = dict(S_less=torch.empty(sh["G"], dtype=torch.complex128, device="cuda"),
               S_gtr=torch.empty(sh["G"], dtype=torch.complex128, device="cuda"),
               P_less=torch.empty(sh["D"], dtype=torch.complex128, device="cuda"),
               P_gtr=torch.empty(sh["D"], dtype=torch.complex128, device="cuda"))
    if fused:
        plan.sigma_pi(t["dH"], t["G_less"], t["G_gtr"], t["D_less"], t["D_gtr"], out["S_less"], out["S_gtr"],
                      out["P_less"], out["P_gtr"], sig_scale, pi_scale)
    else:
        plan.sigma(t["dH"], t["G_less"], t["G_gtr"], t["D_less"], t["D_gtr"], out["S_less"], out["S_gtr"], sig_scale)
        plan.pi(t["dH"], t["G_less"], t["G_gtr"], out["P_less"], out["P_gtr"], pi_scale)
    if own:
        torch.cuda.synchronize()
        plan.close()
    return out


# ---------------------------------------------------------------- RGF (include/qt_rgf.h)
def rgf_count_flops(P: int, bnum: int, bs: int) -> dict:
    """Flops of one RGF solve: the executed dense count and the paper's model 8·(26·bnum − 25)·bs³ per point."""
    d = RgfDesc(P, bnum, bs)
    out = (ctypes.c_double * 2)()
    _check(_get_lib().qt_rgf_count_flops(ctypes.byref(d), out), "qt_rgf_count_flops")
    return dict(executed=out[0], paper_model=out[1])


class Rgf:
    """Owns a qt_rgf_plan_t: diagonal blocks of G^R, G^<, G^> of a batch of block-tridiagonal systems (Eq. 1)."""

    def __init__(self, P: int, bnum: int, bs: int, stream=None):
        self.desc = RgfDesc(P, bnum, bs)
        h = ctypes.c_void_p()
        _check(_get_lib().qt_rgf_plan(ctypes.byref(self.desc), _stream(stream), ctypes.byref(h)), "qt_rgf_plan")
        self.h = h

    def solve(self, Ad, Au, Al, Sl, Sg, GR, GL, GG, stream=None):
        _check(_get_lib().qt_rgf_solve(self.h, _ptr(Ad), _ptr(Au) if Au.numel() else None,
                                       _ptr(Al) if Al.numel() else None, _ptr(Sl), _ptr(Sg), _ptr(GR), _ptr(GL),
                                       _ptr(GG), _stream(stream)), "qt_rgf_solve")

    def check(self, stream=None):
        """(point, block) of the first singular pivot block of the last solve, or None."""
        p, b = ctypes.c_int64(-1), ctypes.c_int64(-1)
        rc = _get_lib().qt_rgf_check_info(self.h, _stream(stream), ctypes.byref(p), ctypes.byref(b))
        if rc == QT_OK:
            return None
        if rc == QT_ERR_INVALID_ARG:
            return int(p.value), int(b.value)
        _check(rc, "qt_rgf_check_info")

    def close(self):
        if self.h:
            _get_lib().qt_rgf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def rgf_run(t: dict, plan: Rgf | None = None):
    """G^R, G^<, G^> diagonal blocks for device inputs t (dict of complex128 CUDA tensors, qtgen.rgf layout)."""
    import torch
    P, nb, bs = t["Ad"].shape[0], t["Ad"].shape[1], t["Ad"].shape[2]
    own = plan is None
    plan = Rgf(P, nb, bs) if own else plan
    out = {k: torch.empty_like(t["Ad"]) for k in ("GR", "GL", "GG")}
    plan.solve(t["Ad"], t["Au"], t["Al"], t["Sl"], t["Sg"], out["GR"], out["GL"], out["GG"])
    bad = plan.check()
    if own:
        plan.close()
    if bad is not None:
        raise QTError(f"qt_rgf_solve: singular pivot block {bad[1]} at point {bad[0]}")
    return out
