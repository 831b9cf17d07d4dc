"""Pins for the CPU oracle (no GPU). Each test checks the oracle against something
other than itself: an independent brute force, closed forms, exact invariants.
Readings R1-R19: DESIGN.md §3. Pins P1-P12: SURVEY.md §8(c)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import qtgen
from qtgen import Problem
from tests.helpers import MICROS, inputs, micro, rel_fro

SIG_AX = (-2, -1)
PI_AX = (-2, -1)


# ------------------------------------------------------------------ P1 brute force
@pytest.mark.parametrize("cfg", range(len(MICROS)))
def test_oracle_matches_brute_force(cfg):
    p = micro(**MICROS[cfg])
    inp = inputs(p, seed=100 + cfg)
    for scale in (1.0, 0.37j):
        SL, SG = oracle.sigma(p, inp, scale)
        BL, BG = oracle.brute_sigma(p, inp, scale)
        assert rel_fro(SL, BL, SIG_AX) < 1e-13 and rel_fro(SG, BG, SIG_AX) < 1e-13
        PL, PG = oracle.pi(p, inp, scale)
        QL, QG = oracle.brute_pi(p, inp, scale)
        assert rel_fro(PL, QL, PI_AX) < 1e-13 and rel_fro(PG, QG, PI_AX) < 1e-13


def test_oracle_matches_brute_force_tiny_config():
    p = qtgen.problem("tiny")
    inp = inputs(p)
    SL, SG = oracle.sigma(p, inp)
    BL, BG = oracle.brute_sigma(p, inp)
    assert rel_fro(SL, BL, SIG_AX) < 1e-13 and rel_fro(SG, BG, SIG_AX) < 1e-13


# ------------------------------------------------------------------ P2 integer-exact mode
@pytest.mark.parametrize("cfg", range(len(MICROS)))
def test_integer_mode_bit_exact(cfg):
    p = micro(**MICROS[cfg])
    inp = inputs(p, mode=qtgen.INTEGER, seed=7 + cfg)
    for scale in (1.0, 1j):
        SL, SG = oracle.sigma(p, inp, scale)
        BL, BG = oracle.brute_sigma(p, inp, scale)
        assert np.array_equal(SL, BL) and np.array_equal(SG, BG)
        PL, PG = oracle.pi(p, inp, scale)
        QL, QG = oracle.brute_pi(p, inp, scale)
        assert np.array_equal(PL, QL) and np.array_equal(PG, QG)
        # integer inputs give integer-multiple-of-1/4 outputs (scale in {1, i})
        assert np.array_equal(SL * 4, np.round(SL * 4))


# ------------------------------------------------------------------ P4 zero / linearity
def test_zero_inputs_give_zero():
    p = micro(**MICROS[1])
    inp = inputs(p)
    z = dict(inp, D_less=np.zeros_like(inp["D_less"]), D_gtr=np.zeros_like(inp["D_gtr"]))
    SL, SG = oracle.sigma(p, z)
    assert not SL.any() and not SG.any()
    z = dict(inp, G_less=np.zeros_like(inp["G_less"]), G_gtr=np.zeros_like(inp["G_gtr"]))
    PL, PG = oracle.pi(p, z)
    assert not PL.any() and not PG.any()


def test_sigma_linear_in_D_and_scale():
    p = micro(**MICROS[3])
    i1 = inputs(p, seed=1)
    i2 = inputs(p, seed=2)
    alpha = 0.3 - 1.7j
    mix = dict(i1, D_less=i1["D_less"] + alpha * i2["D_less"], D_gtr=i1["D_gtr"] + alpha * i2["D_gtr"])
    S1 = oracle.sigma(p, i1)
    S2 = oracle.sigma(p, dict(i1, D_less=i2["D_less"], D_gtr=i2["D_gtr"]))
    Sm = oracle.sigma(p, mix)
    for X in range(2):
        assert rel_fro(Sm[X], S1[X] + alpha * S2[X], SIG_AX) < 1e-13
    # the scale is one complex factor applied at the end (R8)
    Sa = oracle.sigma(p, i1, scale=2.5 - 0.5j)
    Sb = oracle.sigma(p, i1, scale=1.0)
    assert rel_fro(Sa[0], (2.5 - 0.5j) * Sb[0], SIG_AX) < 1e-14


def test_pi_bilinear_in_G():
    p = micro(**MICROS[1])
    i1 = inputs(p, seed=1)
    i2 = inputs(p, seed=2)
    # Π^< is linear in G^< (with G^> fixed)
    alpha = -0.4 + 0.9j
    P1 = oracle.pi(p, i1)
    P2 = oracle.pi(p, dict(i1, G_less=i2["G_less"]))
    Pm = oracle.pi(p, dict(i1, G_less=i1["G_less"] + alpha * i2["G_less"]))
    assert rel_fro(Pm[0], P1[0] + alpha * P2[0], PI_AX) < 1e-13


# ------------------------------------------------------------------ P3 D = δ reduction to a plain sandwich
@pytest.mark.parametrize("m0", [0, 1])
def test_delta_D_reduces_to_plain_sandwich(m0):
    p = micro(Na=6, Nb=3, Norb=3, NE=10, Nw=2, Nkz=3, fill=0.8, seed=11, shift0=2)
    inp = inputs(p, dmode=qtgen.DELTA, delta_m=m0)
    SL, SG = oracle.sigma(p, inp, scale=1.0)
    sm = p.shift0 + m0 * p.shift_step
    rev = qtgen.reverse_slots(p.nbr)
    dH, GL, GG = inp["dH"], inp["G_less"], inp["G_gtr"]
    RL = np.zeros_like(SL)
    RG = np.zeros_like(SG)
    for a in range(p.Na):
        for s in range(p.Nb):
            b = p.nbr[a, s]
            if b < 0:
                continue
            r = rev[a, s]
            for i in range(3):
                L, R = dH[a, s, i], dH[b, r, i]
                for e in range(p.NE):
                    if e - sm >= 0:   # D^< = I3 (Dc = I) with G^<(E - ħω)
                        RL[:, e, a] += L @ GL[:, e - sm, b] @ R
                    if e + sm < p.NE:  # emission term of Σ^> uses D^< (R3) with G^>(E + ħω)
                        RG[:, e, a] += L @ GG[:, e + sm, b] @ R
    assert rel_fro(SL, RL, SIG_AX) < 1e-13 and rel_fro(SG, RG, SIG_AX) < 1e-13
    assert not SL[:, :sm].any()   # rows below the first shift are exactly zero (R7)


# ------------------------------------------------------------------ P5 anti-Hermiticity (north_star)
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_sigma_blocks_anti_hermitian(cfg):
    p = micro(**MICROS[cfg])
    inp = inputs(p, seed=50 + cfg)
    for scale, sign in ((0.37j, -1), (1.0, +1)):
        for S in oracle.sigma(p, inp, scale):
            H = np.conj(np.swapaxes(S, -1, -2))
            assert np.abs(S - sign * H).max() <= 1e-13 * max(np.abs(S).max(), 1e-300)


def test_generator_structure_invariants():
    p = micro(**MICROS[1])
    inp = inputs(p)
    G = inp["G_less"]
    assert np.array_equal(G, -np.conj(np.swapaxes(G, -1, -2)))
    rev = qtgen.reverse_slots(p.nbr)
    D, dH = inp["D_gtr"], inp["dH"]
    for a in range(p.Na):
        assert np.array_equal(D[:, :, a, 0], -np.conj(np.swapaxes(D[:, :, a, 0], -1, -2)))
        for s in range(p.Nb):
            b = p.nbr[a, s]
            if b < 0:
                assert not D[:, :, a, s + 1].any() and not dH[a, s].any()
                continue
            r = rev[a, s]
            assert np.array_equal(D[:, :, a, s + 1], -np.conj(np.swapaxes(D[:, :, b, r + 1], -1, -2)))
            assert np.array_equal(dH[a, s], np.conj(np.swapaxes(dH[b, r], -1, -2)))
    gi = inputs(p, mode=qtgen.INTEGER)["dH"]
    assert set(np.unique(gi.real)) <= {-2.0, -1.0, 0.0, 1.0, 2.0}


# ------------------------------------------------------------------ P6 window edges (R7)
def test_zero_padded_energy_embedding_is_exact():
    p = micro(**MICROS[3])
    inp = inputs(p, seed=3)
    pad = p.shift0 + (p.Nw - 1) * p.shift_step
    q = Problem(p.nbr, p.Norb, p.NE + 2 * pad, p.Nw, p.Nkz, shift0=p.shift0)
    emb = dict(inp)
    for k in ("G_less", "G_gtr"):
        g = np.zeros((p.Nkz, p.NE + 2 * pad) + inp[k].shape[2:], dtype=np.complex128)
        g[:, pad:pad + p.NE] = inp[k]
        emb[k] = g
    S = oracle.sigma(p, inp)
    T = oracle.sigma(q, emb)
    for X in range(2):
        assert np.array_equal(T[X][:, pad:pad + p.NE], S[X])
    P = oracle.pi(p, inp)
    Q = oracle.pi(q, emb)
    for X in range(2):
        assert rel_fro(Q[X], P[X], PI_AX) < 1e-14


# ------------------------------------------------------------------ P7 kz covariance (R4, R5)
@pytest.mark.parametrize("cfg", [1, 3])
def test_kz_roll_covariance(cfg):
    p = micro(**MICROS[cfg])
    inp = inputs(p, seed=9)
    rolled = dict(inp, G_less=np.roll(inp["G_less"], 1, axis=0), G_gtr=np.roll(inp["G_gtr"], 1, axis=0))
    S = oracle.sigma(p, inp)
    T = oracle.sigma(p, rolled)
    for X in range(2):
        assert np.array_equal(T[X], np.roll(S[X], 1, axis=0))
    P = oracle.pi(p, inp)
    Q = oracle.pi(p, rolled)
    for X in range(2):
        assert rel_fro(Q[X], P[X], PI_AX) < 1e-14


# ------------------------------------------------------------------ P8 Π self slot (R9)
def test_pi_self_slot_is_sum_of_neighbour_slots():
    p = micro(**MICROS[2])
    inp = inputs(p, seed=4)
    for P in oracle.pi(p, inp):
        self_sum = P[:, :, :, 1:].sum(axis=3)
        assert np.abs(P[:, :, :, 0] - self_sum).max() <= 1e-13 * np.abs(P).max()
        # empty slots are exactly zero (R12)
        for a in range(p.Na):
            for s in range(p.Nb):
                if p.nbr[a, s] < 0:
                    assert not P[:, :, a, s + 1].any()


# ------------------------------------------------------------------ P9 impulse responses (R2, R3, R5, R6)
def _impulse_problem():
    return micro(Na=6, Nb=3, Norb=3, NE=12, Nw=3, Nkz=3, fill=0.9, seed=21, shift0=1)


@pytest.mark.parametrize("term", ["absorption", "emission"])
def test_sigma_impulse(term):
    p = _impulse_problem()
    base = inputs(p, seed=5)
    k0, e0, b0, q0, m0 = 2, 5, int(np.nonzero((p.nbr >= 0).sum(1))[0][0]), 0, 1
    G = np.zeros_like(base["G_less"])
    G[k0, e0, b0] = base["G_less"][k0, e0, b0]
    D = np.zeros_like(base["D_less"])
    D[q0, m0] = base["D_less"][q0, m0]
    Z = np.zeros_like(D)
    inp = dict(base, G_less=G, G_gtr=np.zeros_like(G),
               D_less=D if term == "absorption" else Z, D_gtr=Z if term == "absorption" else D)
    SL, SG = oracle.sigma(p, inp, scale=1.0)
    assert not SG.any()
    h = p.Nkz // 2
    sm = p.shift0 + m0 * p.shift_step
    kz = (k0 + q0 - h) % p.Nkz                    # kz - qz + h ≡ k0
    e = e0 + sm if term == "absorption" else e0 - sm
    rev = qtgen.reverse_slots(p.nbr)
    expect = np.zeros_like(SL)
    dH = base["dH"]
    for a in range(p.Na):
        for s in range(p.Nb):
            if p.nbr[a, s] != b0:
                continue
            r = rev[a, s]
            Dc = D[q0, m0, b0, r + 1] - D[q0, m0, b0, 0] - D[q0, m0, a, 0] + D[q0, m0, a, s + 1]
            if term == "emission":
                Dc = Dc.T
            for i in range(3):
                for j in range(3):
                    expect[kz, e, a] += Dc[i, j] * (dH[a, s, i] @ G[k0, e0, b0] @ dH[b0, r, j])
    assert 0 <= e < p.NE
    assert rel_fro(SL, expect, SIG_AX) < 1e-14
    nz = np.argwhere(np.abs(SL).sum(axis=(-1, -2)) > 0)
    assert {tuple(x[:2]) for x in nz} == {(kz, e)}


def test_pi_impulse():
    p = _impulse_problem()
    base = inputs(p, seed=6)
    a0 = int(np.nonzero((p.nbr >= 0).sum(1))[0][0])
    s0 = int(np.nonzero(p.nbr[a0] >= 0)[0][0])
    b1 = int(p.nbr[a0, s0])
    k0, e0, k1, e1 = 1, 7, 2, 4
    GL = np.zeros_like(base["G_less"])
    GG = np.zeros_like(base["G_gtr"])
    GL[k0, e0, a0] = base["G_less"][k0, e0, a0]
    GG[k1, e1, b1] = base["G_gtr"][k1, e1, b1]
    PL, PG = oracle.pi(p, dict(base, G_less=GL, G_gtr=GG), scale=1.0)
    h = p.Nkz // 2
    qz = (k0 - k1 + h) % p.Nkz          # k0 = k1 + qz - h
    m = (e0 - e1) - p.shift0            # e0 = e1 + s_m
    rev = qtgen.reverse_slots(p.nbr)
    r = rev[a0, s0]
    dH = base["dH"]
    expect = np.array([[np.trace(dH[b1, r, i] @ GL[k0, e0, a0] @ dH[a0, s0, j] @ GG[k1, e1, b1])
                        for j in range(3)] for i in range(3)])
    got = PL[qz, m, a0, s0 + 1]
    assert np.abs(got - expect).max() <= 1e-14 * np.abs(expect).max()
    nz = np.argwhere(np.abs(PL).sum(axis=(-1, -2)) > 0)
    assert {tuple(x) for x in nz} == {(qz, m, a0, s0 + 1), (qz, m, a0, 0)}


# ------------------------------------------------------------------ P10 ≷ relabel
def test_lesser_greater_relabel():
    p = micro(**MICROS[3])
    inp = inputs(p, seed=12)
    sw = dict(inp, G_less=inp["G_gtr"], G_gtr=inp["G_less"], D_less=inp["D_gtr"], D_gtr=inp["D_less"])
    S = oracle.sigma(p, inp)
    T = oracle.sigma(p, sw)
    assert np.array_equal(S[0], T[1]) and np.array_equal(S[1], T[0])
    P = oracle.pi(p, inp)
    Q = oracle.pi(p, sw)
    assert np.array_equal(P[0], Q[1]) and np.array_equal(P[1], Q[0])


# ------------------------------------------------------------------ block API == full API
def test_block_api_matches_full():
    p = micro(**MICROS[1])
    inp = inputs(p, seed=8)
    S = oracle.sigma(p, inp)
    P = oracle.pi(p, inp)
    rng = np.random.default_rng(0)
    sb = np.stack([rng.integers(0, 2, 20), rng.integers(0, p.Nkz, 20), rng.integers(0, p.NE, 20),
                   rng.integers(0, p.Na, 20)], 1)
    out = oracle.sigma_blocks(p, inp, sb)
    for row, o in zip(sb, out):
        assert np.array_equal(o, S[row[0]][row[1], row[2], row[3]])
    pb = np.stack([rng.integers(0, 2, 20), rng.integers(0, p.Nqz, 20), rng.integers(0, p.Nw, 20),
                   rng.integers(0, p.Na, 20), rng.integers(0, p.Nb + 1, 20)], 1)
    out = oracle.pi_blocks(p, inp, pb)
    for row, o in zip(pb, out):
        assert np.array_equal(o, P[row[0]][row[1], row[2], row[3], row[4]])


# ------------------------------------------------------------------ P11 paper flop model (Table 2)
def test_paper_flop_model_reproduces_table2():
    rows = np.loadtxt(__import__("pathlib").Path(__file__).parent / "golden" / "table2_sse_pflop.txt")
    for nk, omen, dace in rows:
        f_omen = oracle.paper_flops_omen(4864, 34, 3, nk, nk, 706, 70, 12) / 1e15
        assert abs(f_omen - omen) < 0.06, (nk, f_omen, omen)
        # printed (+1) ratio is within 1% of the table; the +N3D fit is within 0.03 Pflop (reading R15)
        f_dace1 = oracle.paper_flops_dace(4864, 34, 3, nk, nk, 706, 70, 12, plus=1) / 1e15
        f_dace3 = oracle.paper_flops_dace(4864, 34, 3, nk, nk, 706, 70, 12, plus=3) / 1e15
        assert abs(f_dace1 - dace) / dace < 0.01
        assert abs(f_dace3 - dace) < 0.03


def test_spec_flop_ratio_example():
    # Nqz=3, Nω=70 -> 2NqzNω/(NqzNω+1) = 420/211
    r = oracle.paper_flops_omen(1, 1, 3, 1, 3, 1, 70, 1) / oracle.paper_flops_dace(1, 1, 3, 1, 3, 1, 70, 1)
    assert abs(r - 420 / 211) < 1e-12


# ------------------------------------------------------------------ geometry (input structure)
def test_geometry_pair_counts_and_shells():
    from qtgen.geometry import diamond_positions, neighbor_table
    assert (neighbor_table(2, 1, 1, 4) >= 0).sum() == 42
    assert (neighbor_table(8, 2, 2, 4) >= 0).sum() == 868
    nbr = neighbor_table(6, 3, 3, 34)
    pos = diamond_positions(6, 3, 3)
    # bulk atoms have exactly 4 + 12 + 12 + 6 = 34 neighbours at squared distances 3, 8, 11, 16 (a/4 units)
    full = np.nonzero((nbr >= 0).all(1))[0]
    assert full.size > 0
    a = full[0]
    d = pos[nbr[a]] - pos[a]
    d[:, 2] = (d[:, 2] + 6) % 12 - 6
    d2 = sorted((d * d).sum(1).tolist())
    assert d2 == [3] * 4 + [8] * 12 + [11] * 12 + [16] * 6


# ------------------------------------------------------------------ R6 with shift_step > 1
@pytest.mark.parametrize("step,shift0", [(2, 1), (3, 2)])
def test_shift_step_brute_force_and_impulse(step, shift0):
    """ħω_m/ΔE = shift0 + m·shift_step: the oracle equals the independent scalar brute force, and a single
    G impulse at e0 with a single D frequency m0 lands exactly at e0 ± (shift0 + m0·step) (Σ) / at frequency
    m = (e0 - e1 - shift0) / step (Π)."""
    p = micro(Na=6, Nb=3, Norb=2, NE=16, Nw=3, Nkz=3, fill=0.9, seed=21, shift0=shift0)
    p.shift_step = step
    inp = inputs(p, seed=9)
    SL, SG = oracle.sigma(p, inp, 0.37j)
    BL, BG = oracle.brute_sigma(p, inp, 0.37j)
    assert rel_fro(SL, BL, SIG_AX) < 1e-13 and rel_fro(SG, BG, SIG_AX) < 1e-13
    PL, PG = oracle.pi(p, inp, 1.0)
    QL, QG = oracle.brute_pi(p, inp, 1.0)
    assert rel_fro(PL, QL, PI_AX) < 1e-13 and rel_fro(PG, QG, PI_AX) < 1e-13
    # Σ impulse: absorption term only (D^> = 0), support at E = e0 + s_m0
    k0, e0, q0, m0 = 1, 3, 0, 2
    b0 = int(np.nonzero((p.nbr >= 0).sum(1))[0][0])
    G = np.zeros_like(inp["G_less"])
    G[k0, e0, b0] = inp["G_less"][k0, e0, b0]
    D = np.zeros_like(inp["D_less"])
    D[q0, m0] = inp["D_less"][q0, m0]
    SL, SG = oracle.sigma(p, dict(inp, G_less=G, G_gtr=np.zeros_like(G), D_less=D, D_gtr=np.zeros_like(D)), 1.0)
    h, sm = p.Nkz // 2, shift0 + m0 * step
    nz = {tuple(x[:2]) for x in np.argwhere(np.abs(SL).sum(axis=(-1, -2)) > 0)}
    assert nz == {((k0 + q0 - h) % p.Nkz, e0 + sm)}
    # Π impulse: G^<_a at e0, G^>_b at e1 = e0 - s_m
    a0 = b0
    s0 = int(np.nonzero(p.nbr[a0] >= 0)[0][0])
    b1 = int(p.nbr[a0, s0])
    m1 = 1
    e1 = 2
    e0p = e1 + shift0 + m1 * step
    GL = np.zeros_like(inp["G_less"])
    GG = np.zeros_like(inp["G_gtr"])
    GL[0, e0p, a0] = inp["G_less"][0, e0p, a0]
    GG[0, e1, b1] = inp["G_gtr"][0, e1, b1]
    PL, _ = oracle.pi(p, dict(inp, G_less=GL, G_gtr=GG), 1.0)
    nz = {tuple(x) for x in np.argwhere(np.abs(PL).sum(axis=(-1, -2)) > 0)}
    assert nz == {(h % p.Nkz, m1, a0, s0 + 1), (h % p.Nkz, m1, a0, 0)}
