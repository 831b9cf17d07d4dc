"""torchrun worker for tests/test_multigpu.py: atom-sharded Σ/Π with the NCCL halo exchange vs the
unsharded single-GPU result in the same precision mode (bit-exact in integer mode, <= 1e-12 relative
Frobenius otherwise: only the order of the FP64 atomic neighbour sums differs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch
import torch.distributed as dist

import paper_1912_10024_b200 as qt
import qtgen


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    name = sys.argv[1] if len(sys.argv) > 1 else "small"
    mode = qtgen.INTEGER if (len(sys.argv) > 2 and sys.argv[2] == "integer") else qtgen.RANDOM
    prec = qt.QT_PREC_FP32_MIXED if (len(sys.argv) > 3 and sys.argv[3] == "fp32") else qt.QT_PREC_FP64
    p = qtgen.problem(name)
    full = qtgen.dev_inputs(p, mode)
    ref = qt.run(p, full, 1.0, 1j, precision=prec)          # unsharded reference on this GPU (same precision)
    obj = [qt.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    if len(sys.argv) > 4 and sys.argv[4] == "energy":
        return energy_case(p, full, ref, prec, mode, obj[0], rank, world, name)
    plan = qt.Plan(p, rank=rank, nranks=world, shard=qt.QT_SHARD_ATOM, unique_id=obj[0], precision=prec)
    info = plan.info()
    a_lo, a_hi, w_lo, w_hi = info["a_lo"], info["a_hi"], info["w_lo"], info["w_hi"]
    win = {}
    for k in ("G_less", "G_gtr", "D_less", "D_gtr"):
        w = torch.zeros_like(full[k][:, :, w_lo:w_hi])
        w[:, :, a_lo - w_lo:a_hi - w_lo] = full[k][:, :, a_lo:a_hi]   # owned atoms only; halo from peers
        win[k] = w.contiguous()
    dH = full["dH"][w_lo:w_hi].contiguous()
    plan.halo_exchange(win["G_less"], win["G_gtr"], win["D_less"], win["D_gtr"])
    torch.cuda.synchronize()
    for k in win:
        assert torch.equal(win[k], full[k][:, :, w_lo:w_hi]), f"halo exchange mismatch in {k}"
    nout = a_hi - a_lo
    S_less = torch.empty((p.Nkz, p.NE, nout, p.Norb, p.Norb), dtype=torch.complex128, device="cuda")
    S_gtr = torch.empty_like(S_less)
    P_less = torch.empty((p.Nqz, p.Nw, nout, p.Nb + 1, 3, 3), dtype=torch.complex128, device="cuda")
    P_gtr = torch.empty_like(P_less)
    plan.sigma(dH, win["G_less"], win["G_gtr"], win["D_less"], win["D_gtr"], S_less, S_gtr, 1.0)
    plan.pi(dH, win["G_less"], win["G_gtr"], P_less, P_gtr, 1j)
    torch.cuda.synchronize()
    worst = 0.0
    for got, r in ((S_less, ref["S_less"][:, :, a_lo:a_hi]), (S_gtr, ref["S_gtr"][:, :, a_lo:a_hi]),
                   (P_less, ref["P_less"][:, :, a_lo:a_hi]), (P_gtr, ref["P_gtr"][:, :, a_lo:a_hi])):
        if mode == qtgen.INTEGER:
            assert torch.equal(got, r)
        num = torch.linalg.matrix_norm(got - r)
        den = torch.linalg.matrix_norm(r)
        assert torch.all(num[den == 0] == 0)
        if (den > 0).any():
            worst = max(worst, float((num[den > 0] / den[den > 0]).max()))
    assert worst <= 1e-12, worst
    dist.barrier()
    if rank == 0:
        print(f"mgpu ok: {name} {world} ranks, precision {prec}, halo {info['halo_bytes']/1e6:.1f} MB/rank, "
              f"max rel {worst:.2e}")
    plan.close()
    dist.destroy_process_group()


def _worst(pairs, exact):
    worst = 0.0
    for got, r in pairs:
        if exact:
            assert torch.equal(got, r)
        num = torch.linalg.matrix_norm(got - r)
        den = torch.linalg.matrix_norm(r)
        assert torch.all(num[den == 0] == 0)
        if (den > 0).any():
            worst = max(worst, float((num[den > 0] / den[den > 0]).max()))
    return worst


def energy_case(p, full, ref, prec, mode, uid, rank, world, name):
    """Energy sharding: G≷ windows [ew_lo, ew_hi) with owned energies filled locally and the halo energies
    exchanged over NCCL; Σ for the owned energies, Π all-reduced over the ranks' energy ranges."""
    plan = qt.Plan(p, rank=rank, nranks=world, shard=qt.QT_SHARD_ENERGY, unique_id=uid, precision=prec)
    info = plan.info()
    e_lo, e_hi, ew_lo, ew_hi = info["e_lo"], info["e_hi"], info["ew_lo"], info["ew_hi"]
    win = {}
    for k in ("G_less", "G_gtr"):
        w = torch.zeros_like(full[k][:, ew_lo:ew_hi])
        w[:, e_lo - ew_lo:e_hi - ew_lo] = full[k][:, e_lo:e_hi]
        win[k] = w.contiguous()
    plan.halo_exchange(win["G_less"], win["G_gtr"], full["D_less"], full["D_gtr"])
    torch.cuda.synchronize()
    for k in win:
        assert torch.equal(win[k], full[k][:, ew_lo:ew_hi]), f"energy halo mismatch in {k}"
    S_less = torch.empty((p.Nkz, e_hi - e_lo, p.Na, p.Norb, p.Norb), dtype=torch.complex128, device="cuda")
    S_gtr = torch.empty_like(S_less)
    P_less = torch.empty((p.Nqz, p.Nw, p.Na, p.Nb + 1, 3, 3), dtype=torch.complex128, device="cuda")
    P_gtr = torch.empty_like(P_less)
    plan.sigma(full["dH"], win["G_less"], win["G_gtr"], full["D_less"], full["D_gtr"], S_less, S_gtr, 1.0)
    plan.pi(full["dH"], win["G_less"], win["G_gtr"], P_less, P_gtr, 1j)
    torch.cuda.synchronize()
    worst = _worst([(S_less, ref["S_less"][:, e_lo:e_hi]), (S_gtr, ref["S_gtr"][:, e_lo:e_hi])],
                   mode == qtgen.INTEGER)
    worst = max(worst, _worst([(P_less, ref["P_less"]), (P_gtr, ref["P_gtr"])], mode == qtgen.INTEGER))
    # FP32 mode: the window offsets change where the FP32 K-chunks and accumulation segments start, so the
    # sharded and unsharded results are two FP32-mode answers (each within 1e-5 of the FP64 oracle)
    tol = 1e-12 if prec == qt.QT_PREC_FP64 else 2e-5
    assert worst <= tol, worst
    dist.barrier()
    if rank == 0:
        print(f"mgpu ok: {name} {world} ranks energy-sharded, precision {prec}, energies [{e_lo},{e_hi}) of "
              f"{p.NE}, halo {info['halo_bytes']/1e6:.1f} MB/rank, max rel {worst:.2e}")
    plan.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
