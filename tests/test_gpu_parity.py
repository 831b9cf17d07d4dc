"""GPU parity: the sm_100a path through the C ABI vs the CPU oracle, on identical seeded inputs.

Bar (north_star): max relative Frobenius error per block <= 1e-12 in FP64; bit-exact in integer
mode (pin P2: every partial sum is an exact binary fraction, so any summation order agrees).
Full comparisons at tiny/micro sizes (several tiles, ragged tails, empty slots, edge windows);
sampled blocks + full-coverage properties at the BASELINE sizes in the bench launch configuration.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import qtgen
from qtgen import Problem
from tests.helpers import MICROS, inputs, micro, rel_fro

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1912_10024_b200 as qt  # noqa: E402

TOL = 1e-12
AX = (-2, -1)


def to_dev(inp):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()}


def gpu_run(p, inp, ss=1j, ps=-1j, **kw):
    out = qt.run(p, to_dev(inp), ss, ps, **kw)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def check_full(p, inp, ss=1j, ps=-1j, exact=False, **kw):
    g = gpu_run(p, inp, ss, ps, **kw)
    SL, SG = oracle.sigma(p, inp, ss)
    PL, PG = oracle.pi(p, inp, ps)
    pairs = ((g["S_less"], SL), (g["S_gtr"], SG), (g["P_less"], PL), (g["P_gtr"], PG))
    for got, ref in pairs:
        if exact:
            assert np.array_equal(got, ref)
        else:
            assert rel_fro(got, ref, AX) <= TOL
    return g


# ------------------------------------------------------------------ generator: device == host, bit for bit
@pytest.mark.parametrize("mode", [qtgen.RANDOM, qtgen.INTEGER, qtgen.DELTA, qtgen.PHYSICAL])
def test_device_generator_matches_host(mode):
    for p in (qtgen.problem("tiny"), micro(**MICROS[2])):
        h = qtgen.host_inputs(p, mode if mode != qtgen.DELTA else qtgen.RANDOM,
                              dmode=mode, delta_m=1 % p.Nw)
        d = qtgen.dev_inputs(p, mode if mode != qtgen.DELTA else qtgen.RANDOM, dmode=mode, delta_m=1 % p.Nw)
        for k in h:
            assert np.array_equal(d[k].cpu().numpy(), h[k]), k
    # sub-range fills use global draw indices
    p = qtgen.problem("tiny")
    full = qtgen.host_G(p, qtgen.ID_GL)
    sub = torch.empty((p.Nkz, 7, 5, p.Norb, p.Norb), dtype=torch.complex128, device="cuda")
    qtgen.dev_G(p, qtgen.ID_GL, sub, e_lo=3, e_hi=10, a_lo=4, a_hi=9)
    assert np.array_equal(sub.cpu().numpy(), full[:, 3:10, 4:9])


# ------------------------------------------------------------------ full parity at tiny sizes
@pytest.mark.parametrize("cfg", range(len(MICROS)))
def test_parity_micro(cfg):
    p = micro(**MICROS[cfg])
    check_full(p, inputs(p, seed=300 + cfg))
    check_full(p, inputs(p, mode=qtgen.INTEGER, seed=400 + cfg), ss=1.0, ps=1j, exact=True)


@pytest.mark.parametrize("cfg", range(len(MICROS)))
def test_parity_micro_physical(cfg):
    """The wide-dynamic-range PHYSICAL envelope (qt_gen.h; G≷ spanning 2^20 in magnitude across energies)."""
    p = micro(**MICROS[cfg])
    check_full(p, inputs(p, mode=qtgen.PHYSICAL, seed=350 + cfg))


def test_parity_tiny_config():
    p = qtgen.problem("tiny")
    check_full(p, inputs(p))
    check_full(p, inputs(p, mode=qtgen.INTEGER), ss=1j, ps=1.0, exact=True)


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("prec", [qt.QT_PREC_FP64, qt.QT_PREC_FP32_MIXED])
def test_parity_multichunk_workspace(fused, prec):
    """workspace_limit = 1 byte (clamped to one item's scratch): Σ and Π run as many chunks (the chunk offsets
    cp0 / pp0 / i0 that the BASELINE sizes reach), through the separate and the fused calls."""
    tol = 1e-12 if prec == qt.QT_PREC_FP64 else 1e-5
    for p in (qtgen.problem("tiny"), micro(Na=14, Nb=12, Norb=3, NE=12, Nw=3, Nkz=3, fill=0.9, seed=5)):
        n0 = qt.launch_count()
        g = gpu_run(p, inputs(p, seed=21), fused=fused, workspace_limit=1, precision=prec)
        nl = qt.launch_count() - n0
        assert nl >= 2 * 3 * 3 + 2 * 3 * 2, nl   # >= 3 Σ chunks (3 launches) and 3 Π chunks (2) per X
        SL, SG = oracle.sigma(p, inputs(p, seed=21), 1j)
        PL, PG = oracle.pi(p, inputs(p, seed=21), -1j)
        for got, ref in ((g["S_less"], SL), (g["S_gtr"], SG), (g["P_less"], PL), (g["P_gtr"], PG)):
            assert rel_fro(got, ref, AX) <= tol
        inp = inputs(p, mode=qtgen.INTEGER, seed=22)
        g = gpu_run(p, inp, 1.0, 1j, fused=fused, workspace_limit=1, precision=prec)
        SL, SG = oracle.sigma(p, inp, 1.0)
        PL, PG = oracle.pi(p, inp, 1j)
        for got, ref in ((g["S_less"], SL), (g["S_gtr"], SG), (g["P_less"], PL), (g["P_gtr"], PG)):
            assert np.array_equal(got, ref)


@pytest.mark.parametrize("cfg", range(len(MICROS)))
def test_parity_fused_call(cfg):
    """qt_sse_sigma_pi (one re-layout shared by Σ and Π) == the oracle, like the separate calls."""
    p = micro(**MICROS[cfg])
    check_full(p, inputs(p, seed=700 + cfg), fused=True)
    check_full(p, inputs(p, mode=qtgen.INTEGER, seed=800 + cfg), ss=1.0, ps=1j, exact=True, fused=True)


@pytest.mark.parametrize("Norb", list(range(1, 13)))
def test_parity_norb_sweep(Norb):
    """Every orbital count 1..12 (all n-fragment widths of the Σ kernel, ragged Norb² tails)."""
    p = micro(Na=7, Nb=4, Norb=Norb, NE=13, Nw=3, Nkz=3, fill=0.7, seed=Norb)
    check_full(p, inputs(p, seed=Norb))


@pytest.mark.parametrize("Nw,NE,shift0,Nkz", [(7, 20, 1, 3), (8, 17, 1, 2), (9, 40, 3, 4), (17, 40, 1, 1),
                                              (3, 4, 1, 3), (2, 3, 2, 5)])
def test_parity_window_sweep(Nw, NE, shift0, Nkz):
    """Frequency counts across m-fragment boundaries, NE < 2Nω, shift0 > 1, even/odd/1 Nkz."""
    p = micro(Na=6, Nb=3, Norb=3, NE=NE, Nw=Nw, Nkz=Nkz, fill=0.8, seed=Nw, shift0=shift0)
    check_full(p, inputs(p, seed=Nw + NE))
    check_full(p, inputs(p, mode=qtgen.INTEGER, seed=Nw), ss=1.0, ps=1.0, exact=True)


@pytest.mark.parametrize("Norb,Nw,NE,step", [(2, 128, 150, 1), (10, 100, 110, 1), (3, 43, 100, 3), (9, 89, 100, 1)])
def test_parity_wide_window(Norb, Nw, NE, step):
    """Shift windows up to the supported maximum ((Nω−1)·shift_step + 1 = 128, qt_sse.h): Π's correlation tile
    then has 12..16 column fragments (two pipeline stages instead of three) and Σ's K up to 257 shifts."""
    nbr = qtgen.geometry.random_graph(6, 5, 0.8, Norb)
    p = Problem(nbr, Norb, NE, Nw, 2, shift_step=step, name="wide")
    check_full(p, inputs(p, seed=960 + Norb))
    check_full(p, inputs(p, mode=qtgen.INTEGER, seed=970 + Norb), ss=1.0, ps=1j, exact=True, fused=True)


@pytest.mark.parametrize("step,shift0,Nw,NE", [(2, 1, 4, 20), (3, 2, 5, 30), (2, 3, 7, 12)])
@pytest.mark.parametrize("prec", [qt.QT_PREC_FP64, qt.QT_PREC_FP32_MIXED])
def test_parity_shift_step(step, shift0, Nw, NE, prec):
    """ħω_m/ΔE = shift0 + m·shift_step with shift_step > 1 (reading R6 generalized): the Σ coefficient
    tables hold zeros between the phonon shifts and the Π correlation computes every shift column and keeps
    the phonon ones."""
    p = micro(Na=6, Nb=3, Norb=3, NE=NE, Nw=Nw, Nkz=3, fill=0.8, seed=step + Nw, shift0=shift0)
    p.shift_step = step
    tol = 1e-12 if prec == qt.QT_PREC_FP64 else 1e-5
    inp = inputs(p, seed=31 + step)
    g = gpu_run(p, inp, precision=prec, fused=True)
    SL, SG = oracle.sigma(p, inp, 1j)
    PL, PG = oracle.pi(p, inp, -1j)
    for got, ref in ((g["S_less"], SL), (g["S_gtr"], SG), (g["P_less"], PL), (g["P_gtr"], PG)):
        assert rel_fro(got, ref, AX) <= tol
    inp = inputs(p, mode=qtgen.INTEGER, seed=41 + step)
    g = gpu_run(p, inp, 1.0, 1j, precision=prec)
    SL, SG = oracle.sigma(p, inp, 1.0)
    PL, PG = oracle.pi(p, inp, 1j)
    for got, ref in ((g["S_less"], SL), (g["S_gtr"], SG), (g["P_less"], PL), (g["P_gtr"], PG)):
        assert np.array_equal(got, ref)


def test_parity_isolated_atoms_and_many_pairs():
    """Atoms with no neighbours (Σ = 0, Π = 0) and atoms with > 8 pairs (several work items)."""
    nbr = qtgen.geometry.random_graph(14, 12, 0.9, 5)
    nbr[0, :] = -1
    for a in range(1, 14):
        nbr[a][nbr[a] == 0] = -1
    p = Problem(nbr, 3, 12, 3, 3)
    g = check_full(p, inputs(p, seed=77))
    assert not g["S_less"][:, :, 0].any() and not g["P_gtr"][:, :, 0].any()
    assert (p.nbr >= 0).sum(1).max() > 8


@pytest.mark.parametrize("Norb,NE,Nw,shift0,step,Nkz,seed", [(9, 13, 3, 1, 1, 3, 2), (10, 21, 5, 2, 1, 2, 3),
                                                             (11, 17, 4, 1, 2, 1, 2), (10, 8, 4, 1, 1, 4, 3),
                                                             (11, 23, 7, 3, 1, 2, 3), (9, 12, 2, 1, 3, 2, 2)])
def test_parity_energy_pair_tiles(Norb, NE, Nw, shift0, step, Nkz, seed):
    """k_sigma_pair (FP64, Norb 9-11): source atoms of 5..12 pairs give items of 4..8 pairs on the energy-pair
    tiles and 1..3-pair remainders on k_sigma in the same chunk (the coefficient / Gt offsets between the two
    launches); odd and even NE (the last pair's E+1 past the window), shift0 / shift_step > 1, Nkz 1..4; the
    separate and fused calls, many chunks with energy sub-ranges (workspace_limit = 1), the deterministic
    neighbour sum; random inputs at 1e-12 and integer inputs bit-exact."""
    nbr = qtgen.geometry.random_graph(16, 13, 0.6, seed)
    deg = (nbr >= 0).sum(1)
    assert (deg >= 4).any() and ((deg % 8 > 0) & (deg % 8 < 4)).any()
    p = Problem(nbr, Norb, NE, Nw, Nkz, shift0=shift0, shift_step=step, name="pair")
    check_full(p, inputs(p, seed=900 + Norb))
    check_full(p, inputs(p, mode=qtgen.INTEGER, seed=910 + Norb), ss=1.0, ps=1j, exact=True, fused=True)
    check_full(p, inputs(p, seed=920 + Norb), fused=True, workspace_limit=1)
    check_full(p, inputs(p, mode=qtgen.INTEGER, seed=930 + Norb), ss=1j, ps=1.0, exact=True,
               flags=qt.QT_FLAG_DETERMINISTIC, workspace_limit=1)


@pytest.mark.parametrize("prec", [qt.QT_PREC_FP64, qt.QT_PREC_FP32_MIXED])
def test_deterministic_flag_bitwise_reproducible(prec):
    """QT_FLAG_DETERMINISTIC: the Σ neighbour sum runs in one fixed order (no floating-point atomics), so two runs
    on random inputs agree bit for bit; the result still meets the parity bar (also with many chunks)."""
    tol = 1e-12 if prec == qt.QT_PREC_FP64 else 1e-5
    for p, ws in ((qtgen.problem("tiny"), 0), (micro(Na=14, Nb=12, Norb=3, NE=12, Nw=3, Nkz=3, fill=0.9, seed=5), 1)):
        inp = inputs(p, seed=61)
        a = gpu_run(p, inp, precision=prec, flags=qt.QT_FLAG_DETERMINISTIC, workspace_limit=ws, fused=True)
        b = gpu_run(p, inp, precision=prec, flags=qt.QT_FLAG_DETERMINISTIC, workspace_limit=ws, fused=True)
        for k in a:
            assert np.array_equal(a[k], b[k]), k
        SL, SG = oracle.sigma(p, inp, 1j)
        assert rel_fro(a["S_less"], SL, AX) <= tol and rel_fro(a["S_gtr"], SG, AX) <= tol
        g = gpu_run(p, inputs(p, mode=qtgen.INTEGER, seed=62), 1.0, 1j, precision=prec,
                    flags=qt.QT_FLAG_DETERMINISTIC)
        SL, SG = oracle.sigma(p, inputs(p, mode=qtgen.INTEGER, seed=62), 1.0)
        assert np.array_equal(g["S_less"], SL) and np.array_equal(g["S_gtr"], SG)


@pytest.mark.slow
def test_deterministic_flag_cfg3_sampled():
    """The deterministic Σ at full cfg3 size: two runs bitwise equal on sampled blocks, and within 1e-12 of the
    default (atomic) path."""
    p = qtgen.problem("cfg3")
    t = qtgen.dev_inputs(p, qtgen.RANDOM)
    outs = [qt.run(p, t, 1j, -1j, flags=qt.QT_FLAG_DETERMINISTIC, fused=True) for _ in range(2)]
    ref = qt.run(p, t, 1j, -1j, fused=True)
    torch.cuda.synchronize()
    for k in ("S_less", "S_gtr"):
        assert torch.equal(outs[0][k], outs[1][k])
        num = torch.linalg.matrix_norm(outs[0][k] - ref[k])
        den = torch.linalg.matrix_norm(ref[k])
        assert float((num[den > 0] / den[den > 0]).max()) <= TOL


def test_calls_on_two_streams_are_ordered():
    """qt_sse_sigma on one stream and qt_sse_pi on another share the plan's scratch: the plan orders them (each call
    waits for the previous call's completion event when the stream changes)."""
    p = micro(Na=14, Nb=12, Norb=3, NE=12, Nw=3, Nkz=3, fill=0.9, seed=5)
    inp = inputs(p, seed=81)
    t = to_dev(inp)
    ref = gpu_run(p, inp)
    plan = qt.Plan(p, workspace_limit=1)   # many chunks: long, overlapping-prone call sequences
    sh = p.shapes()
    out = {k: torch.empty(sh["G" if k[0] == "S" else "D"], dtype=torch.complex128, device="cuda")
           for k in ("S_less", "S_gtr", "P_less", "P_gtr")}
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        plan.sigma(t["dH"], t["G_less"], t["G_gtr"], t["D_less"], t["D_gtr"], out["S_less"], out["S_gtr"], 1j, s1)
        plan.pi(t["dH"], t["G_less"], t["G_gtr"], out["P_less"], out["P_gtr"], -1j, s2)
    torch.cuda.synchronize()
    plan.close()
    for k in out:
        assert rel_fro(out[k].cpu().numpy(), ref[k], AX) <= 1e-13


def test_outputs_overwritten_not_accumulated():
    p = micro(**MICROS[1])
    inp = inputs(p, seed=5)
    t = to_dev(inp)
    plan = qt.Plan(p)
    a = qt.run(p, t, plan=plan)
    b = qt.run(p, t, plan=plan)
    torch.cuda.synchronize()
    for k in a:
        assert rel_fro(b[k].cpu().numpy(), a[k].cpu().numpy(), AX) <= 1e-14
    plan.close()


def test_execute_host_matches_device_path():
    p = micro(**MICROS[3])
    inp = inputs(p, seed=8)
    g = gpu_run(p, inp)
    plan = qt.Plan(p)
    sh = p.shapes()
    o = {k: np.empty(sh["G" if k[0] == "S" else "D"], dtype=np.complex128)
         for k in ("S_less", "S_gtr", "P_less", "P_gtr")}
    c = {k: np.ascontiguousarray(v) for k, v in inp.items()}
    plan.execute_host(c["dH"], c["G_less"], c["G_gtr"], c["D_less"], c["D_gtr"], o["S_less"], o["S_gtr"],
                      o["P_less"], o["P_gtr"])
    for k in o:
        assert rel_fro(o[k], g[k], AX) <= 1e-14
    plan.close()


# ------------------------------------------------------------------ BASELINE sizes: sampled blocks + properties
def _sample_sigma_blocks(p, n, rng):
    deg = (p.nbr >= 0).sum(1)
    surface = np.nonzero(deg < p.Nb)[0]
    bulk = np.nonzero(deg == p.Nb)[0]
    atoms = np.concatenate([rng.choice(surface, n // 2), rng.choice(bulk if bulk.size else surface, n - n // 2)])
    edge = np.concatenate([rng.integers(0, p.Nw + 1, n // 3), rng.integers(p.NE - p.Nw - 1, p.NE, n // 3)])
    es = np.concatenate([edge, rng.integers(0, p.NE, n - edge.size)])
    es = np.clip(es, 0, p.NE - 1)
    return np.stack([rng.integers(0, 2, n), rng.integers(0, p.Nkz, n), es, atoms], 1)


def _sample_pi_blocks(p, n, rng):
    a = rng.integers(0, p.Na, n)
    slots = np.array([rng.choice(np.concatenate([[0], 1 + np.nonzero(p.nbr[x] >= 0)[0]])) for x in a])
    m = np.concatenate([[0, p.Nw - 1], rng.integers(0, p.Nw, n - 2)])
    return np.stack([rng.integers(0, 2, n), rng.integers(0, p.Nqz, n), m, a, slots], 1)


def _sampled_parity(p, mode, n_sig, n_pi, exact):
    rng = np.random.default_rng(2024)
    inp = qtgen.host_inputs(p, mode)
    t = to_dev(inp)
    ss, ps = (1j, -1j) if mode == qtgen.RANDOM else (1.0, 1j)
    out = qt.run(p, t, ss, ps)
    del t
    sb = _sample_sigma_blocks(p, n_sig, rng)
    pb = _sample_pi_blocks(p, n_pi, rng)
    ref_s = oracle.sigma_blocks(p, inp, sb, ss)
    ref_p = oracle.pi_blocks(p, inp, pb, ps)
    S = (out["S_less"], out["S_gtr"])
    P = (out["P_less"], out["P_gtr"])
    got_s = np.stack([S[x][k, e, a].cpu().numpy() for x, k, e, a in sb])
    got_p = np.stack([P[x][q, m, a, s].cpu().numpy() for x, q, m, a, s in pb])
    if exact:
        assert np.array_equal(got_s, ref_s) and np.array_equal(got_p, ref_p)
    else:
        assert rel_fro(got_s, ref_s, AX) <= TOL
        assert rel_fro(got_p, ref_p, AX) <= TOL
    return out


def test_small_config_sampled_random():
    _sampled_parity(qtgen.problem("small"), qtgen.RANDOM, 96, 96, exact=False)


def test_small_config_sampled_integer():
    _sampled_parity(qtgen.problem("small"), qtgen.INTEGER, 96, 96, exact=True)


def test_prof_sampled_physical():
    """PHYSICAL envelope at the cfg3 per-atom shape (Nb = 34, four ∇H shells, Norb 10, NE 176, Nω 70)."""
    _sampled_parity(qtgen.problem("prof"), qtgen.PHYSICAL, 64, 64, exact=False)


@pytest.mark.slow
def test_small_config_full_oracle():
    """BASELINE 'small' nanowire slice, EVERY Σ and Π block against the full oracle (≈16 Tflop of plain-loop
    oracle work), through the fused call in the bench launch configuration (default workspace)."""
    p = qtgen.problem("small")
    check_full(p, qtgen.host_inputs(p, qtgen.RANDOM), fused=True)


@pytest.mark.slow
def test_cfg3_sampled_random():
    """Si FinFET 4,864 atoms, Nb=34, NE=176, Nω=70, Nkz=3: the bench workload and launch configuration."""
    _sampled_parity(qtgen.problem("cfg3"), qtgen.RANDOM, 40, 64, exact=False)


@pytest.mark.slow
def test_cfg3_sampled_integer_bit_exact():
    """Integer-exact inputs at full cfg3 size: sampled blocks must equal the oracle bit for bit (pin P2),
    which checks every index map and the 3M recombination in the bench launch configuration."""
    _sampled_parity(qtgen.problem("cfg3"), qtgen.INTEGER, 24, 48, exact=True)


@pytest.mark.slow
def test_cfg3_delta_full_coverage():
    """P3 at full size: D = δ reduces Σ to plain ∇H·G·∇H sandwiches, checked over EVERY block with cuBLAS."""
    p = qtgen.problem("cfg3")
    m0 = 5
    t = qtgen.dev_inputs(p, qtgen.RANDOM, dmode=qtgen.DELTA, delta_m=m0)
    out = qt.run(p, t, 1.0, -1j)
    sm = p.shift0 + m0
    rev = qtgen.reverse_slots(p.nbr)
    nb = torch.from_numpy(p.nbr.astype(np.int64)).cuda()
    rv = torch.from_numpy(rev.astype(np.int64)).cuda()
    RL = torch.zeros_like(out["S_less"])
    RG = torch.zeros_like(out["S_gtr"])
    dH = t["dH"]
    for s in range(p.Nb):
        valid = nb[:, s] >= 0
        a_idx = torch.nonzero(valid).squeeze(1)
        b_idx = nb[a_idx, s]
        r_idx = rv[a_idx, s]
        for i in range(3):
            L = dH[a_idx, s, i]                       # [n, Norb, Norb]
            R = dH[b_idx, r_idx, i]
            GL = t["G_less"][:, :p.NE - sm][:, :, b_idx]          # E - sm >= 0 rows
            RL[:, sm:, a_idx] += L @ GL @ R
            GG = t["G_gtr"][:, sm:][:, :, b_idx]
            RG[:, :p.NE - sm, a_idx] += L @ GG @ R
    for got, ref in ((out["S_less"], RL), (out["S_gtr"], RG)):
        num = torch.linalg.matrix_norm(got - ref)
        den = torch.linalg.matrix_norm(ref)
        assert torch.all(num[den == 0] == 0)
        assert float((num[den > 0] / den[den > 0]).max()) <= TOL
