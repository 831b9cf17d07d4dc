"""Synthetic Si-FinFET-shaped neighbour graphs (input structure only).

The paper's devices are diamond-lattice Si slices, periodic along z
(PAPER.md P:171-180), with N_b = 34 neighbours per atom for the FinFETs
 and N_b = 4 for the tight-binding-like run.
34 = the first four diamond shells (4 + 12 + 12 + 6); 4 = the first shell.

Coordinates are integers in units of a/4 (a = 0.5431 nm). The conventional
cubic cell holds 8 atoms. Cells nx*ny*nz; x (transport) and y are open, z is
periodic with period 4*nz (minimum image). Atoms are sorted by (x, y, z); the
neighbour slots of an atom are sorted by (distance^2, atom index). Empty slots
(surface atoms) hold -1 (reading R12).
"""
from __future__ import annotations

import numpy as np

# squared shell radii in (a/4)^2 units: shells 1..4 of the diamond lattice
SHELL_D2 = (3, 8, 11, 16)
SHELLS_FOR_NB = {4: 1, 16: 2, 28: 3, 34: 4}

_BASIS = np.array([(0, 0, 0), (0, 2, 2), (2, 0, 2), (2, 2, 0),
                   (1, 1, 1), (1, 3, 3), (3, 1, 3), (3, 3, 1)], dtype=np.int64)


def diamond_positions(nx: int, ny: int, nz: int) -> np.ndarray:
    cells = np.array([(i, j, k) for i in range(nx) for j in range(ny) for k in range(nz)], dtype=np.int64)
    pos = (cells[:, None, :] * 4 + _BASIS[None, :, :]).reshape(-1, 3)
    order = np.lexsort((pos[:, 2], pos[:, 1], pos[:, 0]))
    return pos[order]


def neighbor_table(nx: int, ny: int, nz: int, Nb: int) -> np.ndarray:
    """int32 [Na][Nb] neighbour table, -1 = empty slot."""
    if Nb not in SHELLS_FOR_NB:
        raise ValueError(f"Nb must be one of {sorted(SHELLS_FOR_NB)}")
    cut = SHELL_D2[SHELLS_FOR_NB[Nb] - 1]
    pos = diamond_positions(nx, ny, nz)
    Na = pos.shape[0]
    Lz = 4 * nz
    if 2 * 4 > Lz and Nb == 34:
        raise ValueError("z period too short for the 4th shell (need nz >= 2)")
    nbr = np.full((Na, Nb), -1, dtype=np.int32)
    for a in range(Na):
        d = pos - pos[a]
        d[:, 2] = (d[:, 2] + Lz // 2) % Lz - Lz // 2  # minimum image along periodic z
        d2 = (d * d).sum(axis=1)
        cand = np.nonzero((d2 > 0) & (d2 <= cut))[0]
        cand = cand[np.lexsort((cand, d2[cand]))]
        if cand.size > Nb:
            raise RuntimeError(f"atom {a} has {cand.size} > Nb neighbours")
        nbr[a, :cand.size] = cand
    check_symmetric(nbr)
    return nbr


def check_symmetric(nbr: np.ndarray) -> None:
    Na, Nb = nbr.shape
    for a in range(Na):
        row = nbr[a][nbr[a] >= 0]
        if len(set(row.tolist())) != row.size or (row == a).any():
            raise ValueError(f"bad neighbour row {a}")
        for b in row:
            if a not in nbr[b]:
                raise ValueError(f"asymmetric neighbour relation {a}->{b}")


def reverse_slots(nbr: np.ndarray) -> np.ndarray:
    """rev[a][s] = r with nbr[b][r] == a (b = nbr[a][s]); -1 for empty slots."""
    Na, Nb = nbr.shape
    rev = np.full_like(nbr, -1)
    for a in range(Na):
        for s in range(Nb):
            b = nbr[a, s]
            if b >= 0:
                rev[a, s] = int(np.nonzero(nbr[b] == a)[0][0])
    return rev


def random_graph(Na: int, Nb: int, fill: float, seed: int) -> np.ndarray:
    """Small random symmetric neighbour graph with empty slots, for edge-case tests."""
    rng = np.random.default_rng(seed)
    nbr = np.full((Na, Nb), -1, dtype=np.int32)
    deg = np.zeros(Na, dtype=np.int64)
    pairs = [(a, b) for a in range(Na) for b in range(a + 1, Na)]
    rng.shuffle(pairs)
    for a, b in pairs:
        if deg[a] < Nb and deg[b] < Nb and rng.random() < fill:
            nbr[a, deg[a]] = b
            nbr[b, deg[b]] = a
            deg[a] += 1
            deg[b] += 1
    # shuffle slot order (with holes) per row to exercise arbitrary slot layouts
    for a in range(Na):
        rng.shuffle(nbr[a])
    check_symmetric(nbr)
    return nbr


# BASELINE.json configs -> (cells, Nb, Norb, NE, Nw, Nkz)
CONFIGS = {
    "tiny":  dict(cells=(2, 1, 1), Nb=4, Norb=4, NE=32, Nw=4, Nkz=3),
    "small": dict(cells=(8, 2, 2), Nb=4, Norb=10, NE=256, Nw=16, Nkz=3),
    "cfg3":  dict(cells=(38, 4, 4), Nb=34, Norb=10, NE=176, Nw=70, Nkz=3),
    "cfg3_nb4": dict(cells=(38, 4, 4), Nb=4, Norb=10, NE=176, Nw=70, Nkz=3),
    # the paper's own FinFET orbital count (Norb = 12; Table 2's OMEN row) on the cfg3 slice
    "cfg3_norb12": dict(cells=(38, 4, 4), Nb=34, Norb=12, NE=176, Nw=70, Nkz=3),
    # profiling slice: cfg3's per-atom shape (Nb=34, NE=176, Nω=70, Nkz=3) on 384 atoms
    "prof":  dict(cells=(3, 4, 4), Nb=34, Norb=10, NE=176, Nw=70, Nkz=3),
    "cfg4":  dict(cells=(38, 4, 4), Nb=34, Norb=10, NE=706, Nw=70, Nkz=7),
    # cfg4 / cfg5 per-atom shapes (longest contraction: K = Nqz·(2Nω+1)) on the 384-atom slice
    "prof4": dict(cells=(3, 4, 4), Nb=34, Norb=10, NE=706, Nw=70, Nkz=7),
    "prof5": dict(cells=(3, 4, 4), Nb=34, Norb=10, NE=1000, Nw=70, Nkz=5),
    "cfg5":  dict(cells=(40, 8, 4), Nb=34, Norb=10, NE=1000, Nw=70, Nkz=5),
}
