"""Small end-to-end cases for compute-sanitizer (one process, tiny sizes): FP64 + FP32 (separate and fused calls,
multi-chunk workspace, deterministic flag), a loopback 2x2 grid rank, shift_step 2, and the RGF solver.
usage: compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1912_10024_b200 as qt
import qtgen
from qtgen import rgf as grgf
from tests.helpers import micro

p = qtgen.problem("tiny")
t = qtgen.dev_inputs(p)
for prec in (qt.QT_PREC_FP64, qt.QT_PREC_FP32_MIXED):
    for fused in (False, True):
        qt.run(p, t, precision=prec, fused=fused)
    qt.run(p, t, precision=prec, fused=True, workspace_limit=1, flags=qt.QT_FLAG_DETERMINISTIC)
    # loopback rank 1 of a 2 x 2 grid (atom + energy windows, Π partial)
    plan = qt.Plan(p, rank=1, nranks=4, shard=qt.QT_SHARD_2D, grid_atoms=2, precision=prec)
    i = plan.info()
    w, ew = slice(i["w_lo"], i["w_hi"]), slice(i["ew_lo"], i["ew_hi"])
    win = {k: t[k][:, ew, w].contiguous() for k in ("G_less", "G_gtr")}
    win.update({k: t[k][:, :, w].contiguous() for k in ("D_less", "D_gtr")})
    nout, neo = i["a_hi"] - i["a_lo"], i["e_hi"] - i["e_lo"]
    S = [torch.empty((p.Nkz, neo, nout, p.Norb, p.Norb), dtype=torch.complex128, device="cuda") for _ in range(2)]
    P = [torch.empty((p.Nqz, p.Nw, nout, p.Nb + 1, 3, 3), dtype=torch.complex128, device="cuda") for _ in range(2)]
    plan.sigma_pi(t["dH"][w].contiguous(), win["G_less"], win["G_gtr"], win["D_less"], win["D_gtr"], S[0], S[1], P[0], P[1])
    torch.cuda.synchronize()
    plan.close()
m = micro(Na=6, Nb=3, Norb=3, NE=20, Nw=4, Nkz=3, fill=0.8, seed=3)
m.shift_step = 2
qt.run(m, qtgen.dev_inputs(m), fused=True)
r = grgf.RgfProblem(P=2, bnum=3, bs=24)
qt.rgf_run({k: torch.from_numpy(v).cuda() for k, v in grgf.host_inputs(r).items()})
torch.cuda.synchronize()
print("sanitize case done")
