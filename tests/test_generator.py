"""CPU checks of the input generator's PHYSICAL mode (include/qt_gen.h; SURVEY.md §8(d) "Modes").

The envelope is fixed by its definition in qt_gen.h, so each test checks a property a slip in gen_host.c would
break: exact anti-Hermiticity (a wrong sign or a swapped A_rc / A_cr), a positive semi-definite spectral
function A (a wrong conjugation in X X†), the occupation ladder f / g = 2^-t with t = floor(40 e / NE) - 20
(a wrong energy index or exponent sign), and the shell scaling of ∇H (1 / 0.3 / 0.1 / 0.03 by owner slot)
with ∇H_ba = ∇H_ab† kept exact. Not a parity test of the method: no Eq. 3 / 4 arithmetic lives here.
"""
from __future__ import annotations

import numpy as np

import qtgen


def _herm(x):
    return np.conj(np.swapaxes(x, -1, -2))


def test_physical_G_structure():
    p = qtgen.problem("tiny")
    GL = qtgen.host_G(p, qtgen.ID_GL, qtgen.PHYSICAL)
    GG = qtgen.host_G(p, qtgen.ID_GG, qtgen.PHYSICAL)
    # exactly anti-Hermitian, like every G the kernels consume (R-readings of P:386-389)
    assert np.array_equal(GL, -_herm(GL)) and np.array_equal(GG, -_herm(GG))
    # G< = i f A and G> = -i g A with f + g = 1: A = -i (G< - G>) is Hermitian PSD with the block's X X† / Norb
    A = -1j * (GL - GG)
    ev = np.linalg.eigvalsh(0.5 * (A + _herm(A)).reshape(-1, p.Norb, p.Norb))
    assert ev.min() > -1e-12 * ev.max()
    # the ladder: |G<| / |G>| = f / g = 2^-t per energy, t = floor(40 e / NE) - 20
    nl = np.linalg.norm(GL, axis=(-2, -1))
    ng = np.linalg.norm(GG, axis=(-2, -1))
    for e in range(p.NE):
        t = (40 * e) // p.NE - 20
        np.testing.assert_allclose(nl[:, e] / ng[:, e], 2.0 ** -t, rtol=1e-14)
    # dynamic range actually spans ~2^20 in G<
    assert nl.max() / nl.min() > 2.0 ** 18


def test_physical_G_matches_its_definition():
    """One block rebuilt in Python from the counter the header documents (splitmix64 of seed ^ id·φ ^ index)."""
    p = qtgen.problem("tiny")
    k, e, a = 1, 7, 2
    GL = qtgen.host_G(p, qtgen.ID_GL, qtgen.PHYSICAL)[k, e, a]

    def sm64(z):
        m = (1 << 64) - 1
        z = (z + 0x9E3779B97F4A7C15) & m
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
        return z ^ (z >> 31)

    def draw(idx):
        z = sm64(qtgen.SEED ^ ((qtgen.ID_GL * 0x9E3779B97F4A7C15) & ((1 << 64) - 1)) ^ idx)
        return (z >> 11) * 2.0 ** -53 * 2.0 - 1.0

    nn = p.Norb * p.Norb
    base = ((k * p.NE + e) * p.Na + a) * nn
    X = np.array([[draw(2 * (base + r * p.Norb + c)) + 1j * draw(2 * (base + r * p.Norb + c) + 1)
                   for c in range(p.Norb)] for r in range(p.Norb)])
    A = X @ _herm(X) / p.Norb
    t = (40 * e) // p.NE - 20
    f = 1.0 / (1.0 + 2.0 ** t)
    np.testing.assert_allclose(GL, 1j * f * A, rtol=0, atol=1e-15 * np.abs(A).max())


def test_physical_dH_shells():
    p = qtgen.problem("prof")                        # Nb = 34: four diamond shells 4 / 12 / 12 / 6
    r = qtgen.host_dH(p, qtgen.RANDOM)
    ph = qtgen.host_dH(p, qtgen.PHYSICAL)
    rev = qtgen.reverse_slots(p.nbr)
    scale = np.array([1.0] * 4 + [0.3] * 12 + [0.1] * 12 + [0.03] * 6)
    for a in range(p.Na):
        for s in range(p.Nb):
            b = p.nbr[a, s]
            if b < 0:
                assert not ph[a, s].any()
                continue
            owner = s if a < b else rev[a, s]
            np.testing.assert_allclose(ph[a, s], scale[owner] * r[a, s], rtol=1e-15, atol=0)
            assert np.array_equal(ph[a, s], _herm(ph[b, rev[a, s]]))


def test_physical_D_is_random_mode():
    p = qtgen.problem("tiny")
    for tid in (qtgen.ID_DL, qtgen.ID_DG):
        assert np.array_equal(qtgen.host_D(p, tid, qtgen.PHYSICAL), qtgen.host_D(p, tid, qtgen.RANDOM))
