"""Atom sharding (N > 1) host logic, on CPU with a world_size-2 gloo process group.

Each rank asks the library (host-only qt_sse_shard_info) for its owned atoms and input window, runs the
CPU oracle on the window sub-problem (window-local neighbour table, window slices of the inputs), and the
owned outputs are all-gathered: they must equal the single-process oracle exactly. This checks that the
owned slabs partition the atoms, that every window holds all neighbours its owned atoms read (Eq. 3/4),
and the window <-> global index bookkeeping the GPU path uses.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import qtgen
from qtgen import Problem


def _window_problem(p, w_lo, w_hi):
    nbr = p.nbr[w_lo:w_hi].copy()
    inside = (nbr >= w_lo) & (nbr < w_hi)
    nbr = np.where(inside, nbr - w_lo, -1).astype(np.int32)
    # halo atoms lose their out-of-window neighbours; keep the table symmetric by also dropping
    # the reverse entries (they only affect halo outputs, which are discarded)
    for a in range(nbr.shape[0]):
        for s in range(nbr.shape[1]):
            b = nbr[a, s]
            if b >= 0 and a not in nbr[b]:
                nbr[a, s] = -1
    return Problem(nbr, p.Norb, p.NE, p.Nw, p.Nkz, Nqz=p.Nqz, shift0=p.shift0)


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1912_10024_b200 as qt
    import torch
    p = qtgen.problem("tiny")
    inp = qtgen.host_inputs(p, qtgen.INTEGER)
    info = qt.shard_info(p, rank, world)
    a_lo, a_hi, w_lo, w_hi = info["a_lo"], info["a_hi"], info["w_lo"], info["w_hi"]
    wp = _window_problem(p, w_lo, w_hi)
    # owned atoms keep every neighbour inside the window
    assert (wp.nbr[a_lo - w_lo:a_hi - w_lo] >= 0).sum() == (p.nbr[a_lo:a_hi] >= 0).sum()
    win = {"dH": inp["dH"][w_lo:w_hi], "G_less": inp["G_less"][:, :, w_lo:w_hi], "G_gtr": inp["G_gtr"][:, :, w_lo:w_hi],
           "D_less": inp["D_less"][:, :, w_lo:w_hi], "D_gtr": inp["D_gtr"][:, :, w_lo:w_hi]}
    SL, SG = oracle.sigma(wp, win, 1.0)
    PL, PG = oracle.pi(wp, win, 1j)
    own = slice(a_lo - w_lo, a_hi - w_lo)
    parts = [torch.from_numpy(np.ascontiguousarray(x[:, :, own])).view(torch.float64).reshape(-1)
             for x in (SL, SG, PL, PG)]
    mine = torch.cat(parts)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([mine.numel()]))
    bufs = [torch.zeros(int(s.item()), dtype=torch.float64) for s in sizes]
    if len(set(int(s.item()) for s in sizes)) == 1:
        dist.all_gather(bufs, mine)
    else:
        bufs = [None] * world
        dist.all_gather_object(bufs, mine)
    ranges = [None] * world
    dist.all_gather_object(ranges, (a_lo, a_hi, info["halo_bytes"]))
    if rank == 0:
        result_q.put((ranges, [b.numpy() for b in bufs]))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2])
def test_atom_sharding_matches_single_process_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    ranges, bufs = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=600)
        assert pr.exitcode == 0
    p = qtgen.problem("tiny")
    inp = qtgen.host_inputs(p, qtgen.INTEGER)
    SL, SG = oracle.sigma(p, inp, 1.0)
    PL, PG = oracle.pi(p, inp, 1j)
    # owned slabs partition [0, Na) in order; every rank has a halo to receive
    assert ranges[0][0] == 0 and ranges[-1][1] == p.Na
    assert all(ranges[r][1] == ranges[r + 1][0] for r in range(world - 1))
    assert all(r[2] > 0 for r in ranges)
    for (a_lo, a_hi, _), buf in zip(ranges, bufs):
        ref = np.concatenate([np.ascontiguousarray(x[:, :, a_lo:a_hi]).view(np.float64).ravel()
                              for x in (SL, SG, PL, PG)])
        assert np.array_equal(buf, ref)   # integer mode: bit-exact


def _eworker(rank, world, port, result_q):
    """Energy sharding (the paper's T_E tiling): the oracle on this rank's energy window reproduces the owned
    energies of Σ exactly; the owned energies partition [0, NE); windows are owned ± Dmax."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1912_10024_b200 as qt
    p = qtgen.problem("tiny")
    inp = qtgen.host_inputs(p, qtgen.INTEGER)
    info = qt.shard_info(p, rank, world, shard=qt.QT_SHARD_ENERGY)
    e_lo, e_hi, ew_lo, ew_hi = info["e_lo"], info["e_hi"], info["ew_lo"], info["ew_hi"]
    dmax = p.shift0 + p.Nw - 1
    assert ew_lo == max(0, e_lo - dmax) and ew_hi == min(p.NE, e_hi + dmax)
    assert info["a_lo"] == 0 and info["a_hi"] == p.Na
    wp = Problem(p.nbr, p.Norb, ew_hi - ew_lo, p.Nw, p.Nkz, Nqz=p.Nqz, shift0=p.shift0)
    win = dict(inp)
    win["G_less"] = inp["G_less"][:, ew_lo:ew_hi]
    win["G_gtr"] = inp["G_gtr"][:, ew_lo:ew_hi]
    SL, SG = oracle.sigma(wp, win, 1.0)
    own = slice(e_lo - ew_lo, e_hi - ew_lo)
    mine = [np.ascontiguousarray(SL[:, own]), np.ascontiguousarray(SG[:, own])]
    objs = [None] * world
    dist.all_gather_object(objs, (e_lo, e_hi, info["halo_bytes"], mine))
    if rank == 0:
        result_q.put(objs)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_energy_sharding_matches_single_process_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_eworker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    objs = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=600)
        assert pr.exitcode == 0
    p = qtgen.problem("tiny")
    inp = qtgen.host_inputs(p, qtgen.INTEGER)
    SL, SG = oracle.sigma(p, inp, 1.0)
    assert objs[0][0] == 0 and objs[-1][1] == p.NE
    assert all(objs[r][1] == objs[r + 1][0] for r in range(world - 1))
    assert all(o[2] > 0 for o in objs)
    for e_lo, e_hi, _, (sl, sg) in objs:
        assert np.array_equal(sl, SL[:, e_lo:e_hi]) and np.array_equal(sg, SG[:, e_lo:e_hi])


@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_per_rank_flops_partition_the_total(nranks):
    """qt_sse_shard_info: the ranks' algorithmic flops add up to the unsharded count for both partitions
    (atoms: owned pairs; energies: owned (E, shift) pairs and sandwiches)."""
    import paper_1912_10024_b200 as qt
    p = qtgen.problem("small")
    f = qt.count_flops(p)
    for shard in (qt.QT_SHARD_ATOM, qt.QT_SHARD_ENERGY):
        infos = [qt.shard_info(p, r, nranks, shard=shard) for r in range(nranks)]
        tot = sum(i["flops_sigma"] + i["flops_pi"] for i in infos)
        assert abs(tot - f["total"]) <= 1e-9 * f["total"], (shard, tot, f["total"])
        if shard == qt.QT_SHARD_ENERGY:
            assert [i["e_lo"] for i in infos][0] == 0 and infos[-1]["e_hi"] == p.NE
            assert all(infos[r]["e_hi"] == infos[r + 1]["e_lo"] for r in range(nranks - 1))


def test_energy_pair_kernel_flop_share():
    """qt_sse_shard_info.flops_sigma_pair: in FP64 pair mode (Norb 9..11) every Σ item runs on k_sigma_pair, so its
    share is the whole Σ D-contraction (rank shares included); FP32 mode and Norb outside 9..11 report 0."""
    import paper_1912_10024_b200 as qt
    for name, share in (("small", 1.0), ("prof", 1.0), ("tiny", 0.0)):   # tiny: Norb 4
        p = qtgen.problem(name)
        contr = qt.count_flops(p)["sigma_contraction"]
        i = qt.shard_info(p, 0, 1)
        assert abs(i["flops_sigma_pair"] - share * contr) <= 1e-9 * contr, (name, i["flops_sigma_pair"], contr)
        assert qt.shard_info(p, 0, 1, precision=qt.QT_PREC_FP32_MIXED)["flops_sigma_pair"] == 0.0
    p = qtgen.problem("prof")
    parts = [qt.shard_info(p, r, 3)["flops_sigma_pair"] for r in range(3)]
    tot = qt.count_flops(p)["sigma_contraction"]
    assert abs(sum(parts) - tot) <= 1e-9 * tot


def _gworker(rank, world, ga, port, result_q):
    """Ta x TE grid (the paper's 2-D tiling): the oracle on this rank's window (atom window x energy
    window) reproduces its owned Σ block; Π of the rank is its partial sum over its OWN energies (emulated here by
    zeroing the G^Y_b energies the rank does not own), and the partials of a slab's TE ranks add up to Π."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1912_10024_b200 as qt
    p = qtgen.problem("tiny")
    inp = qtgen.host_inputs(p, qtgen.INTEGER)
    # loopback geometry (no communicator: Π output = the partial of the whole slab)
    i = qt.shard_info(p, rank, world, shard=qt.QT_SHARD_2D, grid_atoms=ga)
    assert (i["Ta"], i["TE"]) == (ga, world // ga) and i["ta"] * i["TE"] + i["te"] == rank
    w_lo, w_hi, ew_lo, ew_hi = i["w_lo"], i["w_hi"], i["ew_lo"], i["ew_hi"]
    wp = _window_problem(p, w_lo, w_hi)
    wp = Problem(wp.nbr, p.Norb, ew_hi - ew_lo, p.Nw, p.Nkz, Nqz=p.Nqz, shift0=p.shift0)
    win = {"dH": inp["dH"][w_lo:w_hi]}
    for k in ("G_less", "G_gtr"):
        win[k] = np.ascontiguousarray(inp[k][:, ew_lo:ew_hi, w_lo:w_hi])
    for k in ("D_less", "D_gtr"):
        win[k] = np.ascontiguousarray(inp[k][:, :, w_lo:w_hi])
    SL, SG = oracle.sigma(wp, win, 1.0)
    own_a = slice(i["a_lo"] - w_lo, i["a_hi"] - w_lo)
    own_e = slice(i["e_lo"] - ew_lo, i["e_hi"] - ew_lo)
    mask = np.zeros(ew_hi - ew_lo, dtype=bool)
    mask[own_e] = True
    part = {}
    for X, (gx, gy) in enumerate((("G_less", "G_gtr"), ("G_gtr", "G_less"))):
        w2 = dict(win)
        w2[gy] = np.where(mask[None, :, None, None, None], win[gy], 0)   # G^Y_b(E): own energies only
        PL, PG = oracle.pi(wp, w2, 1j)
        part[X] = (PL, PG)[X][:, :, own_a]
    objs = [None] * world
    dist.all_gather_object(objs, (i["a_lo"], i["a_hi"], i["e_lo"], i["e_hi"], SL[:, own_e, own_a], SG[:, own_e, own_a],
                                  part[0], part[1]))
    if rank == 0:
        result_q.put(objs)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,ga", [(4, 2), (6, 3)])
def test_2d_grid_matches_single_process_oracle(world, ga):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gworker, args=(r, world, ga, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    objs = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=600)
        assert pr.exitcode == 0
    p = qtgen.problem("tiny")
    inp = qtgen.host_inputs(p, qtgen.INTEGER)
    SL, SG = oracle.sigma(p, inp, 1.0)
    PL, PG = oracle.pi(p, inp, 1j)
    cov = np.zeros((p.NE, p.Na), dtype=np.int64)
    PLs, PGs = np.zeros_like(PL), np.zeros_like(PG)
    for a_lo, a_hi, e_lo, e_hi, sl, sg, pl, pg in objs:
        assert np.array_equal(sl, SL[:, e_lo:e_hi, a_lo:a_hi]) and np.array_equal(sg, SG[:, e_lo:e_hi, a_lo:a_hi])
        PLs[:, :, a_lo:a_hi] += pl
        PGs[:, :, a_lo:a_hi] += pg
        cov[e_lo:e_hi, a_lo:a_hi] += 1
    assert (cov == 1).all()
    assert np.array_equal(PLs, PL) and np.array_equal(PGs, PG)   # integer mode: exact


@pytest.mark.parametrize("cfg,shard,nranks,ga", [("tiny", "2d", 4, 2), ("small", "energy", 3, 0),
                                                 ("small", "2d", 8, 2), ("small", "atom", 5, 0)])
def test_pi_sub_slabs_tile_the_atoms(cfg, shard, nranks, ga):
    """With a communicator, the Π outputs [pa_lo, pa_hi) of all ranks tile [0, Na) once; owned blocks tile
    (energies x atoms) once."""
    import paper_1912_10024_b200 as qt
    p = qtgen.problem(cfg)
    sh = {"atom": qt.QT_SHARD_ATOM, "energy": qt.QT_SHARD_ENERGY, "2d": qt.QT_SHARD_2D}[shard]
    infos = [qt.shard_info(p, r, nranks, shard=sh, grid_atoms=ga) for r in range(nranks)]
    pa = np.zeros(p.Na, dtype=np.int64)
    blk = np.zeros((p.NE, p.Na), dtype=np.int64)
    for i in infos:
        pa[i["pa_lo"]:i["pa_hi"]] += 1
        blk[i["e_lo"]:i["e_hi"], i["a_lo"]:i["a_hi"]] += 1
        assert i["w_lo"] <= i["a_lo"] <= i["a_hi"] <= i["w_hi"] and i["ew_lo"] <= i["e_lo"] <= i["e_hi"] <= i["ew_hi"]
    assert (pa == 1).all() and (blk == 1).all()


@pytest.mark.slow
@pytest.mark.parametrize("cfg,shard,nranks,ga", [("cfg4", "energy", 2, 0), ("cfg4", "energy", 4, 0),
                                                 ("cfg4", "energy", 8, 0), ("cfg4", "atom", 8, 0),
                                                 ("cfg5", "energy", 8, 0), ("cfg5", "atom", 8, 0),
                                                 ("cfg5", "2d", 8, 2)])
def test_north_star_configs_fit_per_rank(cfg, shard, nranks, ga):
    """BASELINE cfg4 (energy-sharded at 2/4/8 B200) and cfg5 (8 B200) fit in HBM: the per-rank footprint the
    library reports (caller window tensors + outputs + plan workspace of 8 GiB, halo staging, Π partial
    buffers, G sum planes) is <= 170 GB of the B200's 180 GB on every rank."""
    import paper_1912_10024_b200 as qt
    p = qtgen.problem(cfg)
    sh = {"atom": qt.QT_SHARD_ATOM, "energy": qt.QT_SHARD_ENERGY, "2d": qt.QT_SHARD_2D}[shard]
    worst = max(qt.shard_info(p, r, nranks, shard=sh, grid_atoms=ga, workspace_limit=8 << 30)["mem_bytes"]
                for r in range(nranks))
    assert worst <= 170e9, f"{cfg} {shard} x{nranks}: {worst / 1e9:.1f} GB per rank"
