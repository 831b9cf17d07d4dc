"""torchrun worker for tests/test_multigpu.py: the sharded path over real NCCL vs the unsharded single-GPU
result in the same precision mode.

Each rank fills ONLY its owned block of the window inputs (the halo region is NaN), so the result can only be
right if the library's exchange delivered every halo entry. Σ is owner-computed; Π sums over energies, so with
TE > 1 each rank receives the reduced sum for its sub-slab [pa_lo, pa_hi). Bit-exact in integer mode; FP64
within 1e-12 (only the order of the floating-point neighbour / energy sums differs); FP32 mode within 2e-5 of
the unsharded FP32 answer (two FP32-mode answers, each within 1e-5 of the FP64 oracle).

usage: mgpu_worker.py CONFIG MODE PREC SHARD [GRID_ATOMS] [CALL]   (CALL: fused | separate)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
import torch.distributed as dist

import paper_1912_10024_b200 as qt
import qtgen


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


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    name, mode_s, prec_s, shard_s = sys.argv[1:5]
    ga = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    call = sys.argv[6] if len(sys.argv) > 6 else "fused"
    mode = qtgen.INTEGER if mode_s == "integer" else qtgen.RANDOM
    prec = qt.QT_PREC_FP32_MIXED if prec_s == "fp32" else qt.QT_PREC_FP64
    shard = {"atom": qt.QT_SHARD_ATOM, "energy": qt.QT_SHARD_ENERGY, "2d": qt.QT_SHARD_2D}[shard_s]
    p = qtgen.problem(name)
    full = qtgen.dev_inputs(p, mode)
    ref = qt.run(p, full, 1.0, 1j, precision=prec)          # unsharded reference on this GPU (same precision)
    obj = [qt.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    plan = qt.Plan(p, rank=rank, nranks=world, shard=shard, grid_atoms=ga, unique_id=obj[0], precision=prec)
    i = plan.info()
    w, ew = slice(i["w_lo"], i["w_hi"]), slice(i["ew_lo"], i["ew_hi"])
    own_a = slice(i["a_lo"] - i["w_lo"], i["a_hi"] - i["w_lo"])
    own_e = slice(i["e_lo"] - i["ew_lo"], i["e_hi"] - i["ew_lo"])
    win = {}
    for k in ("G_less", "G_gtr"):
        t = torch.full_like(full[k][:, ew, w], float("nan"))
        t[:, own_e, own_a] = full[k][:, i["e_lo"]:i["e_hi"], i["a_lo"]:i["a_hi"]]
        win[k] = t.contiguous()
    for k in ("D_less", "D_gtr"):
        t = torch.full_like(full[k][:, :, w], float("nan"))
        t[:, :, own_a] = full[k][:, :, i["a_lo"]:i["a_hi"]]
        win[k] = t.contiguous()
    dH = full["dH"][w].contiguous()
    nout, neo, npa = i["a_hi"] - i["a_lo"], i["e_hi"] - i["e_lo"], i["pa_hi"] - i["pa_lo"]
    c = torch.complex128
    S_less = torch.empty((p.Nkz, neo, nout, p.Norb, p.Norb), dtype=c, device="cuda")
    S_gtr = torch.empty_like(S_less)
    P_less = torch.empty((p.Nqz, p.Nw, npa, p.Nb + 1, 3, 3), dtype=c, device="cuda")
    P_gtr = torch.empty_like(P_less)
    for rep in range(2):   # twice: the second call reuses the plan, its streams, events and partial buffers
        if call == "fused":
            plan.sigma_pi(dH, win["G_less"], win["G_gtr"], win["D_less"], win["D_gtr"], S_less, S_gtr, P_less, P_gtr,
                          1.0, 1j)
        else:
            plan.halo_exchange(win["G_less"], win["G_gtr"], win["D_less"], win["D_gtr"])
            plan.sigma(dH, win["G_less"], win["G_gtr"], win["D_less"], win["D_gtr"], S_less, S_gtr, 1.0)
            plan.pi(dH, win["G_less"], win["G_gtr"], P_less, P_gtr, 1j)
        torch.cuda.synchronize()
    # the halo the library filled is exactly the owners' data
    for k in ("G_less", "G_gtr"):
        assert torch.equal(win[k], full[k][:, ew, w]), f"halo exchange mismatch in {k}"
    for k in ("D_less", "D_gtr"):
        if i["Ta"] > 1:
            assert torch.equal(win[k], full[k][:, :, w]), f"halo exchange mismatch in {k}"
    exact = False
    for nm, got, r in (("S_less", S_less, ref["S_less"][:, i["e_lo"]:i["e_hi"], i["a_lo"]:i["a_hi"]]),
                       ("S_gtr", S_gtr, ref["S_gtr"][:, i["e_lo"]:i["e_hi"], i["a_lo"]:i["a_hi"]]),
                       ("P_less", P_less, ref["P_less"][:, :, i["pa_lo"]:i["pa_hi"]]),
                       ("P_gtr", P_gtr, ref["P_gtr"][:, :, i["pa_lo"]:i["pa_hi"]])):
        num = torch.linalg.matrix_norm(got - r); den = torch.linalg.matrix_norm(r)
        bad = (num > 1e-9 * den.clamp_min(1e-300)) | torch.isnan(num)
        idx = torch.nonzero(bad)
        print(f"rank {rank} {nm}: nbad {int(bad.sum())} of {bad.numel()} nan {int(torch.isnan(got).sum())} "
              f"first {idx[:5].tolist()}", flush=True)
    worst = _worst([(S_less, ref["S_less"][:, i["e_lo"]:i["e_hi"], i["a_lo"]:i["a_hi"]]),
                    (S_gtr, ref["S_gtr"][:, i["e_lo"]:i["e_hi"], i["a_lo"]:i["a_hi"]]),
                    (P_less, ref["P_less"][:, :, i["pa_lo"]:i["pa_hi"]]),
                    (P_gtr, ref["P_gtr"][:, :, i["pa_lo"]:i["pa_hi"]])], exact)
    tol = 1e-12 if prec == qt.QT_PREC_FP64 else 2e-5
    print(f"rank {rank} worst {worst:.3e}", flush=True)
    if worst > tol:
        os._exit(3)
    # the ranks' Π sub-slabs tile the atoms exactly once
    spans = [None] * world
    dist.all_gather_object(spans, (i["pa_lo"], i["pa_hi"]))
    cov = torch.zeros(p.Na, dtype=torch.int64)
    for lo, hi in spans:
        cov[lo:hi] += 1
    assert bool((cov == 1).all()), spans
    dist.barrier()
    if rank == 0:
        print(f"mgpu ok: {name} {world} ranks {shard_s} Ta{i['Ta']} x TE{i['TE']} ({call}), precision {prec}, "
              f"halo {i['halo_bytes'] / 1e6:.1f} MB/rank, Π reduce {i['reduce_bytes'] / 1e6:.1f} MB/rank, "
              f"max rel {worst:.2e}")
    plan.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
