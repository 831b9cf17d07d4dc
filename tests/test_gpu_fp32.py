"""GPU parity of the FP32 mixed-precision mode (QT_PREC_FP32_MIXED) through the C ABI.

In this mode the Σ D-contraction and the Π correlation run on the tcgen05 tensor cores (kind::tf32, every
operand split into two round-to-nearest tf32 terms, FP32 accumulation in TMEM over segments of 128 products:
Σ segments summed in FP32 registers, Π segments in FP64); the ∇H sandwiches run in FP32. Bar (north_star): within 1e-5 relative Frobenius error per block of the FP64
oracle. In integer mode every operand is exact as hi + lo and every partial sum is an integer below 2^24, so
both outputs are bit-exact as well.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import qtgen
from tests.helpers import MICROS, inputs, micro, rel_fro

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1912_10024_b200 as qt  # noqa: E402

TOL_FP32 = 1e-5
TOL_FP64 = 1e-12
AX = (-2, -1)
FP32 = qt.QT_PREC_FP32_MIXED


def _run(p, inp, ss, ps):
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()}
    out = qt.run(p, t, ss, ps, precision=FP32)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def check(p, inp, ss=1j, ps=-1j, exact=False):
    g = _run(p, inp, ss, ps)
    SL, SG = oracle.sigma(p, inp, ss)
    PL, PG = oracle.pi(p, inp, ps)
    for got, ref in ((g["S_less"], SL), (g["S_gtr"], SG)):
        if exact:
            assert np.array_equal(got, ref)
        else:
            assert rel_fro(got, ref, AX) <= TOL_FP32
    for got, ref in ((g["P_less"], PL), (g["P_gtr"], PG)):
        if exact:
            assert np.array_equal(got, ref)
        else:
            assert rel_fro(got, ref, AX) <= TOL_FP32


@pytest.mark.parametrize("cfg", range(len(MICROS)))
def test_fp32_micro(cfg):
    p = micro(**MICROS[cfg])
    check(p, inputs(p, seed=500 + cfg))
    check(p, inputs(p, mode=qtgen.INTEGER, seed=600 + cfg), ss=1.0, ps=1j, exact=True)


def test_fp32_tiny_config():
    p = qtgen.problem("tiny")
    check(p, inputs(p))
    check(p, inputs(p, mode=qtgen.INTEGER), ss=1j, ps=1.0, exact=True)


@pytest.mark.parametrize("Norb", list(range(2, 11)))
def test_fp32_norb_sweep(Norb):
    """Norb 2..10: Norb² = 4..100 of the 128 UMMA rows; ragged coefficient rows (9·npair of 80)."""
    p = micro(Na=7, Nb=4, Norb=Norb, NE=13, Nw=3, Nkz=3, fill=0.7, seed=Norb)
    check(p, inputs(p, seed=Norb))


def test_fp32_norb1_conditioning():
    """Norb = 1: a block is one complex number, and some are sums with heavy cancellation (|Σ| down to
    0.002x the median). Rounding the inputs alone to FP32 already moves those blocks by 5.7e-6 relative
    (oracle on FP32-rounded inputs); FP32 accumulation over the K = Nqz·(2Nω+1) terms adds an absolute error
    of the size of the terms, so the per-block bound here is the conditioning-limited 1e-3 (measured 3.9e-4),
    with the exact-arithmetic check in integer mode."""
    p = micro(Na=7, Nb=4, Norb=1, NE=13, Nw=3, Nkz=3, fill=0.7, seed=1)
    inp = inputs(p, seed=1)
    g = _run(p, inp, 1j, -1j)
    SL, SG = oracle.sigma(p, inp, 1j)
    err = max(rel_fro(g["S_less"], SL, AX), rel_fro(g["S_gtr"], SG, AX))
    print(f"Norb=1 FP32 mode: worst per-block rel. Frobenius error {err:.2e}")
    assert err <= 1e-3
    rel_tensor = np.linalg.norm(g["S_less"] - SL) / np.linalg.norm(SL)
    assert rel_tensor <= TOL_FP32
    check(p, inputs(p, mode=qtgen.INTEGER, seed=1), ss=1.0, ps=1j, exact=True)


@pytest.mark.parametrize("Nw,NE,shift0,Nkz", [(7, 20, 1, 3), (9, 40, 3, 4), (17, 40, 1, 1), (2, 3, 2, 5),
                                              (40, 37, 1, 3)])
def test_fp32_window_sweep(Nw, NE, shift0, Nkz):
    """Every residue of E - Dmax mod 4 (the coefficient delays), windows longer than 32 shifts, NE < 2Nω."""
    p = micro(Na=6, Nb=3, Norb=3, NE=NE, Nw=Nw, Nkz=Nkz, fill=0.8, seed=Nw, shift0=shift0)
    check(p, inputs(p, seed=Nw + NE))
    check(p, inputs(p, mode=qtgen.INTEGER, seed=Nw), ss=1.0, ps=1.0, exact=True)


def test_fp32_unsupported_norb():
    p = micro(Na=5, Nb=3, Norb=11, NE=9, Nw=2, Nkz=3)
    with pytest.raises(qt.QTError, match="status 2"):
        qt.Plan(p, precision=FP32)
    p = micro(Na=5, Nb=3, Norb=2, NE=200, Nw=81, Nkz=3)     # Nω > 80 = the UMMA N of the Π correlation
    with pytest.raises(qt.QTError, match="status 2"):
        qt.Plan(p, precision=FP32)


@pytest.mark.parametrize("cfg", range(len(MICROS)))
def test_fp32_micro_physical(cfg):
    """FP32 mode on the wide-dynamic-range PHYSICAL envelope (qt_gen.h): the per-block bar still holds when
    G≷ magnitudes span 2^20 across the energies a Σ / Π block sums over."""
    p = micro(**MICROS[cfg])
    check(p, inputs(p, mode=qtgen.PHYSICAL, seed=650 + cfg))


def test_fp32_prof_physical_sampled():
    """PHYSICAL envelope at the cfg3 per-atom shape (Nb = 34 with ∇H shells 1 / 0.3 / 0.1 / 0.03), FP32 mode:
    sampled Σ (half at the low- and high-energy ends of the occupation ladder) and Π blocks at 1e-5."""
    p = qtgen.problem("prof")
    inp = qtgen.host_inputs(p, qtgen.PHYSICAL)
    out = _run(p, inp, 1j, -1j)
    rng = np.random.default_rng(9)
    n = 64
    es = np.concatenate([rng.integers(0, 20, n // 4), rng.integers(p.NE - 20, p.NE, n // 4),
                         rng.integers(0, p.NE, n - n // 2)])
    sb = np.stack([rng.integers(0, 2, n), rng.integers(0, p.Nkz, n), es, rng.integers(0, p.Na, n)], 1)
    S = (out["S_less"], out["S_gtr"])
    err_s = rel_fro(np.stack([S[x][k, e, a] for x, k, e, a in sb]), oracle.sigma_blocks(p, inp, sb, 1j), AX)
    a_s = rng.integers(0, p.Na, n)
    pb = np.stack([rng.integers(0, 2, n), rng.integers(0, p.Nqz, n), rng.integers(0, p.Nw, n), a_s,
                   [rng.choice(np.concatenate([[0], 1 + np.nonzero(p.nbr[x] >= 0)[0]])) for x in a_s]], 1)
    P = (out["P_less"], out["P_gtr"])
    err_p = rel_fro(np.stack([P[x][q, m, a, s] for x, q, m, a, s in pb]), oracle.pi_blocks(p, inp, pb, -1j), AX)
    print(f"prof PHYSICAL FP32 mode: max per-block rel. Frobenius error Σ {err_s:.2e}, Π {err_p:.2e}")
    assert err_s <= TOL_FP32 and err_p <= TOL_FP32, (err_s, err_p)


def test_fp32_small_config_sampled():
    p = qtgen.problem("small")
    inp = qtgen.host_inputs(p, qtgen.RANDOM)
    out = _run(p, inp, 1j, -1j)
    rng = np.random.default_rng(7)
    sb = np.stack([rng.integers(0, 2, 64), rng.integers(0, p.Nkz, 64), rng.integers(0, p.NE, 64),
                   rng.integers(0, p.Na, 64)], 1)
    ref = oracle.sigma_blocks(p, inp, sb, 1j)
    S = (out["S_less"], out["S_gtr"])
    got = np.stack([S[x][k, e, a] for x, k, e, a in sb])
    assert rel_fro(got, ref, AX) <= TOL_FP32


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["prof4", "prof5"])
def test_fp32_long_contraction_sampled(cfg):
    """cfg4 / cfg5 per-atom shapes (Nkz = 7 / 5: the longest Σ accumulation, K = Nqz·(2Nω+1) = 987 / 705 products;
    NE = 706 / 1000): sampled Σ and Π blocks within 1e-5 of the FP64 oracle."""
    p = qtgen.problem(cfg)
    inp = qtgen.host_inputs(p, qtgen.RANDOM)
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()}
    out = qt.run(p, t, 1j, -1j, precision=FP32, fused=True)
    del t
    rng = np.random.default_rng(17)
    n = 48
    sb = np.stack([rng.integers(0, 2, n), rng.integers(0, p.Nkz, n), rng.integers(0, p.NE, n),
                   rng.integers(0, p.Na, n)], 1)
    got = np.stack([(out["S_less"], out["S_gtr"])[x][k, e, a].cpu().numpy() for x, k, e, a in sb])
    err_s = rel_fro(got, oracle.sigma_blocks(p, inp, sb, 1j), AX)
    a_s = rng.integers(0, p.Na, n)
    pb = np.stack([rng.integers(0, 2, n), rng.integers(0, p.Nqz, n), rng.integers(0, p.Nw, n), a_s,
                   [1 + rng.choice(np.nonzero(p.nbr[x] >= 0)[0]) for x in a_s]], 1)
    got_p = np.stack([(out["P_less"], out["P_gtr"])[x][q, m, a, s].cpu().numpy() for x, q, m, a, s in pb])
    err_p = rel_fro(got_p, oracle.pi_blocks(p, inp, pb, -1j), AX)
    print(f"{cfg} FP32 mode: max per-block rel. Frobenius error Σ {err_s:.2e}, Π {err_p:.2e}")
    assert err_s <= TOL_FP32 and err_p <= TOL_FP32, (err_s, err_p)


@pytest.mark.slow
def test_fp32_cfg3_sampled():
    """The bench workload (cfg3) in FP32 mode: sampled Σ and Π blocks vs the oracle at 1e-5."""
    p = qtgen.problem("cfg3")
    inp = qtgen.host_inputs(p, qtgen.RANDOM)
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()}
    out = qt.run(p, t, 1j, -1j, precision=FP32)
    del t
    rng = np.random.default_rng(11)
    n = 32
    sb = np.stack([rng.integers(0, 2, n), rng.integers(0, p.Nkz, n),
                   np.concatenate([rng.integers(0, 8, n // 4), rng.integers(0, p.NE, n - n // 4)]),
                   rng.integers(0, p.Na, n)], 1)
    ref = oracle.sigma_blocks(p, inp, sb, 1j)
    S = (out["S_less"], out["S_gtr"])
    got = np.stack([S[x][k, e, a].cpu().numpy() for x, k, e, a in sb])
    err_s = rel_fro(got, ref, AX)
    a_s = rng.integers(0, p.Na, n)
    pb = np.stack([rng.integers(0, 2, n), rng.integers(0, p.Nqz, n),
                   np.concatenate([[0, p.Nw - 1], rng.integers(0, p.Nw, n - 2)]), a_s,
                   [rng.choice(np.concatenate([[0], 1 + np.nonzero(p.nbr[x] >= 0)[0]])) for x in a_s]], 1)
    ref_p = oracle.pi_blocks(p, inp, pb, -1j)
    P = (out["P_less"], out["P_gtr"])
    got_p = np.stack([P[x][q, m, a, s].cpu().numpy() for x, q, m, a, s in pb])
    err_p = rel_fro(got_p, ref_p, AX)
    print(f"cfg3 FP32 mode: max per-block rel. Frobenius error Σ {err_s:.2e}, Π {err_p:.2e}")
    assert err_s <= TOL_FP32 and err_p <= TOL_FP32, (err_s, err_p)
