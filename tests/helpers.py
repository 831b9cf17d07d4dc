"""Shared test helpers: small problems, comparison metrics."""
from __future__ import annotations

import numpy as np

import qtgen
from qtgen import Problem
from qtgen.geometry import random_graph


def micro(Na=5, Nb=3, Norb=2, NE=9, Nw=2, Nkz=3, fill=0.7, seed=1, shift0=1, Nqz=None) -> Problem:
    """Small random symmetric graph with empty slots and shuffled slot order."""
    nbr = random_graph(Na, Nb, fill, seed)
    return Problem(nbr, Norb, NE, Nw, Nkz, Nqz=Nkz if Nqz is None else Nqz, shift0=shift0, name="micro")


# a spread of tiny shapes that exercise sentinels, even/odd Nkz (h = Nkz//2), shift0 > 1, NE = 2Nω
MICROS = [
    dict(Na=4, Nb=2, Norb=2, NE=8, Nw=2, Nkz=1, fill=1.0, seed=3),           # SPEC S:291 shape
    dict(Na=5, Nb=3, Norb=2, NE=9, Nw=2, Nkz=3, fill=0.7, seed=1),
    dict(Na=6, Nb=4, Norb=3, NE=6, Nw=3, Nkz=2, fill=0.6, seed=7),           # NE = 2Nω, even Nkz
    dict(Na=5, Nb=3, Norb=2, NE=11, Nw=3, Nkz=4, fill=0.8, seed=5, shift0=2),
]


def rel_fro(x, ref, axes):
    """Per-block relative Frobenius error over `axes`; blocks with zero reference must be exactly zero."""
    num = np.sqrt((np.abs(x - ref) ** 2).sum(axis=axes))
    den = np.sqrt((np.abs(ref) ** 2).sum(axis=axes))
    zero = den == 0
    assert np.all(num[zero] == 0), "nonzero output where the reference block is exactly zero"
    return float((num[~zero] / den[~zero]).max()) if (~zero).any() else 0.0


def inputs(p, mode=qtgen.RANDOM, seed=qtgen.SEED, **kw):
    return qtgen.host_inputs(p, mode, seed, **kw)
