"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol
include/qt_sse.h declares, validates its arguments, and counts algorithmic flops."""
from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import qtgen
from tests.helpers import micro

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_declared_symbol():
    import paper_1912_10024_b200 as qt
    header = (ROOT / "include" / "qt_sse.h").read_text()
    declared = set(re.findall(r"^(?:qt_status|void|const char\*|uint64_t)\s+(qt_sse_\w+)\s*\(", header, re.M))
    assert declared == set(qt.EXPORTED)
    for name in declared:
        assert hasattr(qt.lib, name), name


def test_library_exports_every_rgf_symbol():
    import paper_1912_10024_b200 as qt
    header = (ROOT / "include" / "qt_rgf.h").read_text()
    declared = set(re.findall(r"^(?:qt_status|void)\s+(qt_rgf_\w+)\s*\(", header, re.M))
    assert declared == set(qt.EXPORTED_RGF)
    for name in declared:
        assert hasattr(qt.lib, name), name


def test_generator_libraries_export_declared_symbols():
    header = (ROOT / "include" / "qt_gen.h").read_text()
    declared = set(re.findall(r"^(?:void|int)\s+(qtgen_\w+)\s*\(", header, re.M))
    assert len(declared) == 6
    host = ctypes.CDLL(str(ROOT / "qtgen" / "libqtgen_host.so"))
    dev = ctypes.CDLL(str(ROOT / "qtgen" / "libqtgen_dev.so"))
    for name in declared:
        lib = host if "_host_" in name else dev
        assert hasattr(lib, name), name


def _count(p):
    import paper_1912_10024_b200 as qt
    return qt.count_flops(p)


def test_flop_count_matches_loop_count():
    """F_alg (qt_sse_count_flops) == direct enumeration of the in-window work."""
    for cfg in (dict(Na=6, Nb=3, Norb=3, NE=10, Nw=3, Nkz=3, fill=0.7, seed=2, shift0=2),
                dict(Na=5, Nb=4, Norb=2, NE=7, Nw=2, Nkz=2, fill=0.9, seed=4)):
        p = micro(**cfg)
        f = _count(p)
        npairs = int((p.nbr >= 0).sum())
        NN = p.Norb ** 2
        sig_c = pi_c = 0
        for e in range(p.NE):
            for m in range(p.Nw):
                sm = p.shift0 + m
                sig_c += (e - sm >= 0) + (e + sm < p.NE)
                pi_c += e + sm < p.NE
        # per X: Nkz*Nqz*pairs*count*9*NN complex MACs, 8 flops each; both X
        assert f["sigma_contraction"] == 2 * p.Nkz * p.Nqz * npairs * sig_c * 9 * NN * 8
        assert f["pi_contraction"] == 2 * p.Nkz * p.Nqz * npairs * pi_c * 9 * NN * 8
        assert f["sigma_sandwich"] == 2 * p.Nkz * p.NE * npairs * 12 * p.Norb ** 3 * 8


def test_flop_count_cfg3():
    """cfg3 (Nb=34) F_alg = 601 Tflop (SURVEY §8(a) totals)."""
    p = qtgen.problem("cfg3")
    f = _count(p)
    assert abs(f["total"] / 1e12 - 601.3) < 1.0
    assert abs(f["sigma_contraction"] / 1e12 - 380.7) < 0.5


def test_invalid_arguments_rejected_before_device_use():
    import paper_1912_10024_b200 as qt
    p = micro(Na=5, Nb=3, Norb=2, NE=9, Nw=2, Nkz=3, fill=0.7, seed=1)
    out = (ctypes.c_double * 4)()
    nbr = np.ascontiguousarray(p.nbr)
    for field, val in (("Na", 0), ("N3D", 2), ("Nqz", 2), ("shift0", 0), ("NE", -1)):
        d = qt.make_desc(p)
        setattr(d, field, val)
        assert qt.lib.qt_sse_count_flops(ctypes.byref(d), nbr.ctypes.data, out) == qt.QT_ERR_INVALID_ARG
        h = ctypes.c_void_p()
        assert qt.lib.qt_sse_plan(ctypes.byref(d), nbr.ctypes.data, None, ctypes.byref(h)) == qt.QT_ERR_INVALID_ARG
        assert not h.value
    # asymmetric / self / out-of-range neighbour tables
    d = qt.make_desc(p)
    for bad in ("asym", "self", "range", "dup"):
        n = nbr.copy()
        a = int(np.nonzero((n >= 0).any(1))[0][0])
        s = int(np.nonzero(n[a] >= 0)[0][0])
        if bad == "asym":
            n[a, s] = -1
        elif bad == "self":
            n[a, s] = a
        elif bad == "range":
            n[a, s] = p.Na
        else:
            free = np.nonzero(n[a] < 0)[0]
            if free.size == 0:
                continue
            n[a, free[0]] = n[a, s]
        assert qt.lib.qt_sse_count_flops(ctypes.byref(d), np.ascontiguousarray(n).ctypes.data, out) == \
            qt.QT_ERR_INVALID_ARG, bad
    # unsupported: Norb > 12; FP32 mixed mode with Norb > 10; an unknown precision
    d = qt.make_desc(p)
    d.Norb = 13
    h = ctypes.c_void_p()
    assert qt.lib.qt_sse_plan(ctypes.byref(d), nbr.ctypes.data, None, ctypes.byref(h)) == qt.QT_ERR_UNSUPPORTED
    d = qt.make_desc(p, precision=qt.QT_PREC_FP32_MIXED)
    d.Norb = 11
    assert qt.lib.qt_sse_plan(ctypes.byref(d), nbr.ctypes.data, None, ctypes.byref(h)) == qt.QT_ERR_UNSUPPORTED
    d = qt.make_desc(p, precision=qt.QT_PREC_FP32_MIXED)
    d.Nw = 81                                      # > 80 = the UMMA N of the FP32-mode Π correlation
    assert qt.lib.qt_sse_plan(ctypes.byref(d), nbr.ctypes.data, None, ctypes.byref(h)) == qt.QT_ERR_UNSUPPORTED
    d = qt.make_desc(p)
    d.precision = 7
    assert qt.lib.qt_sse_plan(ctypes.byref(d), nbr.ctypes.data, None, ctypes.byref(h)) == qt.QT_ERR_UNSUPPORTED
    assert qt.lib.qt_sse_status_string(qt.QT_ERR_UNSUPPORTED) == b"unsupported configuration"
    qt.lib.qt_sse_destroy(None)   # NULL-safe
