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
