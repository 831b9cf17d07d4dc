"""Pins of the RGF oracle (oracle/rgf.py: the dense definition of Eq. 1) against what the
mathematics fixes, not against itself: the residual A·G^R = I, a 2x2 closed form, SPEC's identity-matrix example
(S:229), the Σ^> − Σ^< = Σ^R − Σ^A ⇒ G^> − G^< = G^R − G^A identity, anti-Hermiticity of G^≷,
and point independence. Also checks the C-ABI flop model against the paper's RGF formula."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import rgf as orgf
from qtgen import rgf as grgf


@pytest.mark.parametrize("name", ["rgf_tiny", "rgf_small"])
def test_residual_and_offdiagonal_consistency(name):
    p = grgf.problem(name)
    inp = grgf.host_inputs(p, seed=3)
    GR, GL, GG = orgf.solve(inp)
    for q in range(p.P):
        A = orgf.assemble(inp["Ad"], inp["Au"], inp["Al"], q)
        R = np.linalg.inv(A)
        assert np.abs(A @ R - np.eye(p.N)).max() < 1e-11
        # every diagonal block of the oracle is the corresponding block of a solve with unit right-hand sides
        for n in range(p.bnum):
            rhs = np.zeros((p.N, p.bs), dtype=np.complex128)
            rhs[n * p.bs:(n + 1) * p.bs] = np.eye(p.bs)
            col = np.linalg.solve(A, rhs)[n * p.bs:(n + 1) * p.bs]
            assert np.abs(col - GR[q, n]).max() < 1e-11 * max(1.0, np.abs(col).max())


def test_two_site_closed_form():
    """bnum = 2, bs = 1: A = [[a, b], [c, d]] ⇒ G^R = [[d, −b], [−c, a]] / (ad − bc), G^< = G^R diag(σ0, σ1) G^A."""
    a, b, c, d = 0.7 + 0.2j, -0.3 + 0.1j, -0.3 - 0.1j, -0.4 + 0.05j
    s0, s1 = 0.3j, 0.8j
    inp = dict(Ad=np.array([[[[a]], [[d]]]]), Au=np.array([[[[b]]]]), Al=np.array([[[[c]]]]),
               Sl=np.array([[[[s0]], [[s1]]]]), Sg=np.array([[[[-s1]], [[-s0]]]]))
    GR, GL, GG = orgf.solve(inp)
    det = a * d - b * c
    g = np.array([[d, -b], [-c, a]]) / det
    assert abs(GR[0, 0, 0, 0] - g[0, 0]) < 1e-14 * abs(g[0, 0]) and abs(GR[0, 1, 0, 0] - g[1, 1]) < 1e-14 * abs(g[1, 1])
    gl00 = abs(g[0, 0]) ** 2 * s0 + abs(g[0, 1]) ** 2 * s1
    gl11 = abs(g[1, 0]) ** 2 * s0 + abs(g[1, 1]) ** 2 * s1
    assert abs(GL[0, 0, 0, 0] - gl00) < 1e-14 * abs(gl00) and abs(GL[0, 1, 0, 0] - gl11) < 1e-14 * abs(gl11)


def test_identity_matrix_example():
    """A = I, Σ^< = iI ⇒ G^< = iI."""
    P, nb, bs = 2, 3, 4
    eye = np.broadcast_to(np.eye(bs, dtype=np.complex128), (P, nb, bs, bs)).copy()
    z = np.zeros((P, nb - 1, bs, bs), dtype=np.complex128)
    GR, GL, GG = orgf.solve(dict(Ad=eye, Au=z, Al=z, Sl=1j * eye, Sg=-1j * eye))
    assert np.array_equal(GR, eye) and np.array_equal(GL, 1j * eye)


@pytest.mark.parametrize("name", ["rgf_tiny", "rgf_small"])
def test_lesser_greater_identity_and_antihermiticity(name):
    """With no extra broadening (η = 0) A − A† = −(Σ^R − Σ^A), so G^R − G^A = G^R (Σ^> − Σ^<) G^A = G^> − G^<."""
    p = grgf.problem(name)
    inp = grgf.host_inputs(p, seed=5, eta=0.0)
    GR, GL, GG = orgf.solve(inp)
    GA = np.conj(np.swapaxes(GR, -1, -2))
    scale = np.abs(GR).max()
    assert np.abs((GG - GL) - (GR - GA)).max() < 1e-12 * scale
    for G in (GL, GG):
        assert np.abs(G + np.conj(np.swapaxes(G, -1, -2))).max() < 1e-12 * np.abs(G).max()


def test_points_are_independent():
    p = grgf.problem("rgf_tiny")
    inp = grgf.host_inputs(p, seed=7)
    full = orgf.solve(inp)
    one = orgf.solve(inp, points=[2, 0])
    for a, b in zip(full, one):
        assert np.array_equal(a[[2, 0]], b)


def test_flop_model_matches_paper_formula():
    import paper_1912_10024_b200 as qt
    f = qt.rgf_count_flops(16, 76, 640)
    assert f["paper_model"] == 16 * 8.0 * (26 * 76 - 25) * 640.0 ** 3
    # the executed dense count is the same order (the paper's 26 products per block vs 21 GEMMs + 1 inversion)
    assert 0.7 < f["executed"] / f["paper_model"] < 1.0   # 21 GEMMs + 4/3 for the inversion vs 26
