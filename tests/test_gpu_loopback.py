"""Single-GPU "loopback" parity of the sharded (multi-GPU) path: one process plans every rank of a Ta x TE grid
 WITHOUT a communicator, fills each rank's window halo from the full tensors (what the NCCL
exchange delivers), runs the rank's Σ/Π through the C ABI, and reassembles: Σ blocks are owner-computed, Π
blocks of a rank are its PARTIAL sums over its own energies, summed here over the TE ranks of each
atom slab. The result must equal the CPU oracle element by element — bit-exact in integer mode (pin P2), within
1e-12 per block in FP64 and 1e-5 in the FP32 mixed mode.

This runs on the driver's 1-GPU box, so the sharded kernels (atom windows with Nout < Nwin, energy windows with
E0 != 0, Π partial sums, sub-slab work lists) are covered without a second GPU; the NCCL halo exchange and the
Π reduction themselves are covered by tests/test_multigpu.py (2 GPUs).
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

AX = (-2, -1)
SHARDS = {"atom": qt.QT_SHARD_ATOM, "energy": qt.QT_SHARD_ENERGY, "2d": qt.QT_SHARD_2D}


def loopback(p, inp, shard, nranks, grid_atoms=0, precision=qt.QT_PREC_FP64, fused=True, ss=1j, ps=-1j,
             workspace_limit=0):
    """Σ≷, Π≷ assembled from every rank of the grid, each run through its own loopback plan."""
    full = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()}
    sh = p.shapes()
    S = {k: np.zeros(sh["G"], dtype=np.complex128) for k in ("S_less", "S_gtr")}
    P = {k: np.zeros(sh["D"], dtype=np.complex128) for k in ("P_less", "P_gtr")}
    covered = np.zeros((p.NE, p.Na), dtype=np.int64)
    seen_e0 = set()
    for r in range(nranks):
        plan = qt.Plan(p, rank=r, nranks=nranks, shard=SHARDS[shard], grid_atoms=grid_atoms, precision=precision,
                       workspace_limit=workspace_limit)
        i = plan.info()
        assert i["pa_lo"] == i["a_lo"] and i["pa_hi"] == i["a_hi"]   # loopback: partial Π of the whole slab
        w = slice(i["w_lo"], i["w_hi"])
        ew = slice(i["ew_lo"], i["ew_hi"])
        seen_e0.add(i["e_lo"] - i["ew_lo"])
        win = {k: full[k][:, ew, w].contiguous() for k in ("G_less", "G_gtr")}
        win.update({k: full[k][:, :, w].contiguous() for k in ("D_less", "D_gtr")})
        dH = full["dH"][w].contiguous()
        nout, neo = i["a_hi"] - i["a_lo"], i["e_hi"] - i["e_lo"]
        o = {k: torch.full((p.Nkz, neo, nout, p.Norb, p.Norb), float("nan"), dtype=torch.complex128, device="cuda")
             for k in ("S_less", "S_gtr")}
        o.update({k: torch.full((p.Nqz, p.Nw, nout, p.Nb + 1, 3, 3), float("nan"), dtype=torch.complex128,
                                device="cuda") for k in ("P_less", "P_gtr")})
        if fused:
            plan.sigma_pi(dH, win["G_less"], win["G_gtr"], win["D_less"], win["D_gtr"], o["S_less"], o["S_gtr"],
                          o["P_less"], o["P_gtr"], ss, ps)
        else:
            plan.sigma(dH, win["G_less"], win["G_gtr"], win["D_less"], win["D_gtr"], o["S_less"], o["S_gtr"], ss)
            plan.pi(dH, win["G_less"], win["G_gtr"], o["P_less"], o["P_gtr"], ps)
        torch.cuda.synchronize()
        with pytest.raises(qt.QTError, match="status 2"):   # a loopback plan cannot exchange
            plan.halo_exchange(win["G_less"], win["G_gtr"], win["D_less"], win["D_gtr"])
        plan.close()
        for k in S:
            S[k][:, i["e_lo"]:i["e_hi"], i["a_lo"]:i["a_hi"]] = o[k].cpu().numpy()
        for k in P:
            P[k][:, :, i["a_lo"]:i["a_hi"]] += o[k].cpu().numpy()
        covered[i["e_lo"]:i["e_hi"], i["a_lo"]:i["a_hi"]] += 1
    assert (covered == 1).all(), "the ranks' blocks must tile (energies x atoms) exactly once"
    return S, P, seen_e0


def compare(p, inp, S, P, ss, ps, tol, exact):
    SL, SG = oracle.sigma(p, inp, ss)
    PL, PG = oracle.pi(p, inp, ps)
    worst = 0.0
    for got, ref in ((S["S_less"], SL), (S["S_gtr"], SG), (P["P_less"], PL), (P["P_gtr"], PG)):
        if exact:
            assert np.array_equal(got, ref)
        else:
            worst = max(worst, rel_fro(got, ref, AX))
    assert worst <= tol, worst
    return worst


CASES = [("atom", 2, 0), ("atom", 3, 0), ("energy", 2, 0), ("energy", 3, 0), ("2d", 4, 2), ("2d", 6, 3)]


@pytest.mark.parametrize("shard,nranks,ga", CASES)
def test_loopback_tiny_fp64(shard, nranks, ga):
    p = qtgen.problem("tiny")
    inp = inputs(p, seed=11)
    S, P, e0s = loopback(p, inp, shard, nranks, ga)
    compare(p, inp, S, P, 1j, -1j, 1e-12, False)
    if shard != "atom":
        assert max(e0s) > 0   # energy windows with E0 != 0 were exercised
    S, P, _ = loopback(p, inputs(p, mode=qtgen.INTEGER, seed=12), shard, nranks, ga, ss=1.0, ps=1j, fused=False)
    compare(p, inputs(p, mode=qtgen.INTEGER, seed=12), S, P, 1.0, 1j, 0.0, True)


@pytest.mark.parametrize("shard,nranks,ga", [("atom", 2, 0), ("energy", 3, 0), ("2d", 4, 2)])
def test_loopback_micro_graphs(shard, nranks, ga):
    """Random graphs with empty slots and shuffled slot order; NE = 2Nω; shift0 > 1."""
    for k in (1, 2, 3):
        p = micro(**MICROS[k])
        if p.NE < nranks:
            continue
        inp = inputs(p, mode=qtgen.INTEGER, seed=40 + k)
        S, P, _ = loopback(p, inp, shard, nranks, ga, ss=1.0, ps=1j)
        compare(p, inp, S, P, 1.0, 1j, 0.0, True)


@pytest.mark.parametrize("shard,nranks,ga", [("atom", 2, 0), ("energy", 2, 0), ("2d", 4, 2)])
def test_loopback_tiny_fp32(shard, nranks, ga):
    p = qtgen.problem("tiny")
    inp = inputs(p, seed=13)
    S, P, _ = loopback(p, inp, shard, nranks, ga, precision=qt.QT_PREC_FP32_MIXED)
    compare(p, inp, S, P, 1j, -1j, 1e-5, False)
    inp = inputs(p, mode=qtgen.INTEGER, seed=14)
    S, P, _ = loopback(p, inp, shard, nranks, ga, precision=qt.QT_PREC_FP32_MIXED, ss=1.0, ps=1j)
    compare(p, inp, S, P, 1.0, 1j, 0.0, True)


def test_loopback_multichunk():
    """The smallest workspace: every rank runs many Σ and Π chunks (chunk offsets inside shard windows)."""
    p = qtgen.problem("tiny")
    inp = inputs(p, mode=qtgen.INTEGER, seed=15)
    n0 = qt.launch_count()
    S, P, _ = loopback(p, inp, "2d", 4, 2, ss=1.0, ps=1j, workspace_limit=1)
    assert qt.launch_count() - n0 > 4 * 2 * 3 * 3   # >= 3 Σ chunks per rank and X (3 launches each)
    compare(p, inp, S, P, 1.0, 1j, 0.0, True)


@pytest.mark.parametrize("shard,nranks,ga", [("atom", 4, 0), ("energy", 4, 0), ("2d", 4, 2)])
def test_loopback_small_config(shard, nranks, ga):
    """BASELINE 'small' nanowire slice (Norb=10, NE=256, Nω=16): bit-exact in integer mode for every block."""
    p = qtgen.problem("small")
    inp = qtgen.host_inputs(p, qtgen.INTEGER)
    S, P, _ = loopback(p, inp, shard, nranks, ga, ss=1.0, ps=1j)
    rng = np.random.default_rng(3)
    n = 64
    sb = np.stack([rng.integers(0, 2, n), rng.integers(0, p.Nkz, n), rng.integers(0, p.NE, n),
                   rng.integers(0, p.Na, n)], 1)
    ref = oracle.sigma_blocks(p, inp, sb, 1.0)
    got = np.stack([(S["S_less"], S["S_gtr"])[x][k, e, a] for x, k, e, a in sb])
    assert np.array_equal(got, ref)
    a = rng.integers(0, p.Na, n)
    pb = np.stack([rng.integers(0, 2, n), rng.integers(0, p.Nqz, n), rng.integers(0, p.Nw, n), a,
                   [rng.integers(0, p.Nb + 1) for _ in a]], 1)
    ref = oracle.pi_blocks(p, inp, pb, 1j)
    got = np.stack([(P["P_less"], P["P_gtr"])[x][q, m, aa, s] for x, q, m, aa, s in pb])
    assert np.array_equal(got, ref)
